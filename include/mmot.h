/* mmot.h -- C ABI of the B200-native fast tensor-vector product / multi-marginal Sinkhorn
 * for the L1 pairwise cost on a uniform 1-D grid (arXiv 2405.19246).
 *
 * Citations: P:n = line n of the paper's LaTeX, with section / equation /
 * algorithm.  Notation follows the paper and DESIGN.md:
 *   l marginals, N grid points x_i = x_min + i h, h = (x_max - x_min)/(N-1)
 *   cost c(i) = h sum_{p<q} |i_p - i_q|
 *   kernel K = exp(-C/eta) = lambda^{E(i)}, lambda = e^{-h/eta}
 *   scalings phi_1..phi_l, plan t_i = K_i prod_q phi_q[i_q]
 *   J_k = K x_{q != k} phi_q  (tensor-vector product, mode k free)
 *   k-th marginal of the plan m_k = phi_k * J_k
 *   Sinkhorn update phi_k <- mu_k / J_k, k = 1..l, freshest peers
 *   W = sum_i c(i) t(i) = <phi_l, (C.K) x_{q<l} phi_q>
 *
 * Conventions for every entry point:
 *   - Array arguments of the compute calls are DEVICE pointers owned by the caller,
 *     16-byte aligned, contiguous, element type given by the context dtype (MMOT_F64:
 *     double; MMOT_F32: float) except where stated.  Marginal index k is 0-based.
 *   - All work is enqueued on the context's CUDA stream; calls return without waiting
 *     unless they fill a HOST output (mmot_sinkhorn's report, mmot_cost's W), in which
 *     case they synchronise that stream once at the end.
 *   - Argument errors are detected on the host before any launch.  Data errors (NaN/Inf,
 *     negative or zero mass) are detected on device and reported through mmot_report /
 *     the return value of the synchronising calls.
 *   - A context is not reentrant: one host thread per context at a time.
 *   - No call allocates device memory after mmot_create* except mmot_sinkhorn_host
 *     (staging buffers, allocated once on first use).
 */
#ifndef MMOT_H_
#define MMOT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMOT_VERSION_MAJOR 0
#define MMOT_VERSION_MINOR 1
#define MMOT_MAX_L 8          /* supported marginal counts: 2..MMOT_MAX_L; l = 7, 8 (64 / 128 subset
                               * states) run on the stabilised log-domain family only: MMOT_F64,
                               * MMOT_KERNEL_AUTO or _STABLE, mmot_create / mmot_create_batched;
                               * every other request returns MMOT_EUNSUPPORTED */

#if defined(__GNUC__)
#define MMOT_API __attribute__((visibility("default")))
#else
#define MMOT_API
#endif

typedef struct mmot_ctx mmot_ctx;  /* opaque; owns device workspace only */

typedef enum { MMOT_F64 = 0, MMOT_F32 = 1 } mmot_dtype;

/* Representation of the scaling vectors u[] passed to mmot_marginal / mmot_sinkhorn /
 * mmot_cost / mmot_init_uniform.  MMOT_LOG (default): u[q] holds g_q = log phi_q (the
 * paper's potentials up to sign/scale, Remark 1 P:138-151), -inf allowed.
 * MMOT_LINEAR: u[q] holds phi_q itself.  u[] is always float64 (both dtypes). */
typedef enum { MMOT_LOG = 0, MMOT_LINEAR = 1 } mmot_repr;

typedef enum {
    MMOT_OK = 0,
    MMOT_EINVAL = 1,       /* invalid scalar argument (l, N, eta, grid, k, iters, NULL) */
    MMOT_ESHAPE = 2,       /* pointer / batch / shard layout mismatch                     */
    MMOT_ENONFINITE = 3,   /* NaN or Inf in a marginal or scaling vector                  */
    MMOT_ENEGMASS = 4,     /* negative entry in a marginal                                */
    MMOT_EZEROMASS = 5,    /* a marginal with zero total mass                              */
    MMOT_EOVERFLOW = 6,    /* a product J_k left the representable range (P:1184 analogue) */
    MMOT_ECUDA = 7,        /* CUDA runtime error (see mmot_last_error)                    */
    MMOT_ENCCL = 8,        /* NCCL error (sharded contexts)                               */
    MMOT_ENOMEM = 9,       /* device allocation failed                                    */
    MMOT_EUNSUPPORTED = 10, /* valid request this build does not implement               */
    MMOT_EPRECISION = 11   /* single-walk precision guard tripped on a sharded context     */
} mmot_status;

/* Uniform grid x_i = x_min + i h, i = 0..N-1 (endpoints included, A1). */
typedef struct { double x_min, x_max; } mmot_grid;

/* Kernel family of the single-instance products.
 *   AUTO: single-walk kernels when a chain of >= 64 points satisfies
 *         P * max_a a(l-a) * h/eta <= 1 (large N, small h/eta: e.g. C4), else two-walk.
 *   TWO_WALK: suffix states by a right-to-left walk with TMEM / local checkpoints (any eta).
 *   SINGLE_WALK: suffix states walked forward through the inverse recurrence step (each grid
 *         point read once); l <= 5.  Its rounding error grows like exp(P * max_a a(l-a) h/eta),
 *         so outside the bound above the caller accepts the accuracy loss. */
typedef enum {
    MMOT_KERNEL_AUTO = 0,
    MMOT_KERNEL_TWO_WALK = 1,
    MMOT_KERNEL_SINGLE_WALK = 2,
    MMOT_KERNEL_PERSISTENT = 3, /* one warp per instance, all sweeps in one launch (the batched kernel,
                                   batch = 1); AUTO picks it for l <= 5, N <= 4096, MMOT_F64, chunk = 0 */
    MMOT_KERNEL_STABLE = 4      /* stabilised family (a8): the recurrence in the LOG domain (states carried
                                   as logarithms; the paper's log-domain stabilisation, Remark 1 P:138-151,
                                   Algorithm 5), one warp per instance walking the whole grid:
                                   any eta / dynamic range, O(N) latency per product.  Uniform grids,
                                   single (mmot_create) and batched (mmot_create_batched) contexts.  The
                                   other families fall back to it automatically, see
                                   mmot_stable_fallback_count. */
} mmot_kernel;

typedef struct {
    int check_every;    /* residual cadence in sweeps; 0 = only when tol > 0, every sweep (default) */
    int residual_mode;  /* 0 = paper: sum_{k<l} ||m_k - mu_k||_1 (Alg. 1 line 7, generalised) */
    mmot_repr repr;     /* representation of u[] (default MMOT_LOG) */
    int chunk;          /* grid points per chunk (chain); 0 = automatic */
    mmot_kernel kernel; /* kernel family (default MMOT_KERNEL_AUTO) */
} mmot_opts;

typedef struct {
    int iters_done;     /* sweeps completed (each sweep = l updates) */
    double residual;    /* last computed residual (NaN if never computed) */
    int converged;      /* 1 if residual <= tol stopped the loop */
    int status;         /* mmot_status of the run */
    int fail_iter;      /* sweep index at which EOVERFLOW/ENONFINITE was detected, else -1 */
} mmot_report;

/* Create a context for single instances of (l, N, eta) on `grid`.
 *   l in [2, MMOT_MAX_L], N >= 1, eta > 0 finite, x_max > x_min when N > 1.
 *   dt: element type of the marginals and of mmot_marginal's output (u[] is fp64 for both):
 *       MMOT_F64 double; MMOT_F32 float (fp32 I/O: the scans run in fp64 on widened copies, so an
 *       fp32 context reproduces the fp64 result of the fp32-rounded inputs).
 *   opts may be NULL (defaults).  cuda_stream: cudaStream_t (NULL = legacy default stream).
 * The per-edge weights w_a = lambda^{a(l-a)} = exp(-a(l-a) h/eta), a = 0..l, are computed
 * once in fp64 on the host (A15).  Allocates all workspace.
 * On error *out is set to NULL. */
MMOT_API mmot_status mmot_create(int l, int64_t N, double eta, mmot_grid grid, mmot_dtype dt,
                        const mmot_opts *opts, void *cuda_stream, mmot_ctx **out);

/* Create a context for `batch` independent instances of (l, N) on the same grid, instance b
 * with its own eta_host[b] (BASELINE C5: 8192 x (l=5, N=4096), eta ~ logU[1e-3, 1e-1]).
 *   l in [2, MMOT_MAX_L]: the persistent / pair / CTA families for l <= 5; l = 6..8 on the stabilised
 *   family (MMOT_F64, MMOT_KERNEL_AUTO or _STABLE; EUNSUPPORTED otherwise); N >= 1, batch >= 1, every eta finite > 0;
 *   dt: MMOT_F64 or MMOT_F32 (fp32 I/O, as for mmot_create).  eta_host is copied.
 * Layouts for the compute calls on a batched context: every array argument is a plane of
 * `batch` consecutive N-vectors ([batch][N], instance-major); mmot_cost fills W[batch] (host);
 * mmot_sinkhorn runs at most `iters` sweeps per instance, one warp per instance on device, each
 * instance stopping at its own first residual <= tol (tol > 0; residual every check_every sweeps);
 * the report gives the max sweeps done and max last residual over the instances, converged = all
 * converged, and the first failing instance's status (if any).
 * Internally each instance's scalings carry one exponent per 1/32 of the grid and marginal,
 * so instances whose |log phi| exceeds the fp64 range (eta = 1e-3) stay representable. */
MMOT_API mmot_status mmot_create_batched(int l, int64_t N, int64_t batch, const double *eta_host, mmot_grid grid,
                                         mmot_dtype dt, const mmot_opts *opts, void *cuda_stream, mmot_ctx **out);

/* Non-uniform 1-D grids (the paper's footnote to the uniform-grid assumption, PAPER.md:182;
 * SURVEY §8(f) NEXT-3).  x_host[N]: the grid points, finite and strictly increasing (copied).
 * The L1 cost is c(i) = sum_{p<q} |x[i_p] - x[i_q]|; every grid edge e (between points e-1 and e)
 * gets its own decay lambda_e = exp(-(x[e] - x[e-1]) / eta).  Kernel families: batched contexts
 * and single instances with l <= 5, N <= 4096 (or opts->kernel = MMOT_KERNEL_PERSISTENT) run on the
 * persistent kernel; larger single instances (l in [2, 6]) on the two-walk family
 * (MMOT_KERNEL_SINGLE_WALK -> EUNSUPPORTED; batched contexts accept only AUTO / PERSISTENT).  All
 * other arguments, layouts and the compute calls are those of mmot_create / mmot_create_batched
 * (mmot_cost returns W = sum_i c(i) t(i) in x's units).
 * Errors: EINVAL for a NULL / non-finite / non-increasing x_host, plus those of the uniform
 * constructors. */
MMOT_API mmot_status mmot_create_points(int l, int64_t N, double eta, const double *x_host, mmot_dtype dt,
                                        const mmot_opts *opts, void *cuda_stream, mmot_ctx **out);
MMOT_API mmot_status mmot_create_batched_points(int l, int64_t N, int64_t batch, const double *eta_host,
                                                const double *x_host, mmot_dtype dt, const mmot_opts *opts,
                                                void *cuda_stream, mmot_ctx **out);

/* 2-D grids (§4.1).  An N1 x N2 uniform mesh of
 * [x_min, x_max] x [y_min, y_max] (endpoints included; vertical spacing h1 = (x_max-x_min)/(N1-1),
 * horizontal h2 = (y_max-y_min)/(N2-1)), the L1 cost c = sum_{p<q} (|i1_p - i1_q| h1 + |i2_p - i2_q| h2)
 * and K = lambda1^{E1} lambda2^{E2}.  l = 3 (the paper's 2-D case; other l:
 * EUNSUPPORTED).  Every vector argument of the compute calls is the flattened mesh, COLUMN-MAJOR:
 * x[i1 + N1 i2], N1 N2 elements.  The product is Algorithm 6's structure: an
 * outer recurrence over the N2 columns whose states are column vectors, with six batched 1-D
 * FTVP-1 products per column (grid2d.cu); mmot_cost returns W = <phi_3, (C.K) x phi_1 x phi_2>
 * (the 2-D cost product the paper omits, by dual numbers, A21).
 * Plain fp64 (EOVERFLOW on loss of range); mmot_sinkhorn / mmot_marginal / mmot_cost /
 * mmot_init_uniform (phi = 1/(N1 N2)) as for mmot_create. */
typedef struct { double x_min, x_max, y_min, y_max; } mmot_grid2d;
MMOT_API mmot_status mmot_create_2d(int l, int64_t N1, int64_t N2, double eta, mmot_grid2d grid, mmot_dtype dt,
                                    const mmot_opts *opts, void *cuda_stream, mmot_ctx **out);

/* Create rank `rank`'s part of ONE instance sharded over `world` GPUs by contiguous grid
 * chunks (BASELINE C4 on 1/2/4/8 GPUs).  The rank owns global points
 * [lo, hi) = mmot_shard_range(N_global, rank, world) of every vector; all array arguments of
 * the compute calls are that rank's local chunks (hi - lo elements).  The grid spacing is the
 * global h = (x_max - x_min)/(N_global - 1).  nccl_unique_id: 128 bytes from
 * mmot_nccl_unique_id on one rank, broadcast by the caller (e.g. torch.distributed).  Every
 * rank must make the same sequence of calls (each product performs one ncclAllGather of the
 * whole-shard prefix/suffix operators, ~2 (l) 2^(l-1) doubles per rank; residual and cost one
 * ncclAllReduce of a double).  Returns ENCCL if NCCL cannot be loaded or initialised.
 * Collective consistency: the data checks use the mass of the whole marginal, the status and
 * stop flag are max-reduced over the ranks (after the checks, at every early-exit poll and at the
 * end of a solve), and with tol > 0 the early exit is decided synchronously every 8 sweeps on the
 * agreed flag, so all ranks leave the sweep loop together and report the same status.
 * mmot_init_uniform fills log phi = -log N_global (the global problem's 1/N). */
MMOT_API mmot_status mmot_create_sharded(int l, int64_t N_global, double eta, mmot_grid grid, mmot_dtype dt,
                                         const void *nccl_unique_id, int rank, int world, const mmot_opts *opts,
                                         void *cuda_stream, mmot_ctx **out);

/* Virtual shards: an in-process group of `world` sharded contexts on ONE device, the device-side
 * test mode of the sharded path (SURVEY §4 suite 4).  Each rank's context is created with
 * mmot_create_sharded_virtual and driven by its own host thread on its own CUDA stream; the
 * collectives of mmot_create_sharded (all-gather of the whole-shard operators, all-reduce of the
 * residual / cost / data checks) become a host barrier plus cross-stream event waits and
 * device-to-device copies, so the shard-boundary seeding, the carry composition with real
 * predecessors and the partial reductions run exactly as on `world` GPUs (no kernel waits on
 * another).  world in [1, 16].  The group must outlive its contexts; mmot_vgroup_destroy(NULL) is
 * a no-op.  All ranks must make the same sequence of calls concurrently (a rank that fails to
 * create leaves the others waiting, as with NCCL). */
typedef struct mmot_vgroup mmot_vgroup;
MMOT_API mmot_status mmot_vgroup_create(int world, mmot_vgroup **out);
MMOT_API void mmot_vgroup_destroy(mmot_vgroup *group);
MMOT_API mmot_status mmot_create_sharded_virtual(int l, int64_t N_global, double eta, mmot_grid grid, mmot_dtype dt,
                                                 mmot_vgroup *group, int rank, const mmot_opts *opts,
                                                 void *cuda_stream, mmot_ctx **out);

/* 128-byte NCCL unique id for mmot_create_sharded (host memory). */
MMOT_API mmot_status mmot_nccl_unique_id(void *out);

/* Grid chunk [*lo, *hi) of `rank` out of `world` for N_global points: lo = floor(rank N / world). */
MMOT_API void mmot_shard_range(int64_t N_global, int rank, int world, int64_t *lo, int64_t *hi);

/* Host reference of the carry composition the sharded contexts run on device (no GPU needed):
 * ops_all = [world][2][l 2^(l-1)] gathered whole-shard operators (prefix, suffix; entry
 * G_c[S] at c 2^(l-1) + S, c = 0..l-1, S a subset of the l-1 bound marginals), fin / bin =
 * the 2^(l-1) prefix / suffix states entering shard `rank` from the left / right. */
MMOT_API mmot_status mmot_compose_rank_carries(int l, const double *ops_all, int world, int rank, double *fin,
                                               double *bin);

/* Host reference of the composition sharded contexts run on device for the restricted
 * next-update scan (single-walk Sinkhorn updates, l in 3..5; no GPU needed): elems_all =
 * [world][2][l 2^(l-2)] gathered whole-shard affine elements (prefix, suffix; entry A_c[V] at
 * (c-1) 2^(l-2) + V for c = 1..l-1, offsets at (l-1) 2^(l-2) + U), fin / bin = the 2^(l-2)
 * new-part states entering shard `rank` from the left / right. */
MMOT_API mmot_status mmot_compose_rank_affine(int l, const double *elems_all, int world, int rank, double *fin,
                                              double *bin);

/* m_k = phi_k * J_k(phi_{-k}) -- the k-th marginal of K . (phi_1 x ... x phi_l)
 * (P:1021), computed by the O(N) separated-summation scans.
 *   k in [0, l); u: host array of l device pointers (repr per opts, float64, length N each);
 *   out: device pointer, N elements of the context dtype (linear units).  Asynchronous. */
MMOT_API mmot_status mmot_marginal(mmot_ctx *ctx, int k, const void *const *u, void *out);

/* Generalized Sinkhorn (Algorithm 4): at most `iters` sweeps of the
 * l Gauss-Seidel updates phi_k <- mu_k / J_k; after each sweep whose index is a multiple of
 * check_every, Res = sum_{k<l-1} ||phi_k J_k - mu_k||_1 on the end-of-sweep vectors (P:168
 * generalised, A6); stops after the first sweep with Res <= tol (tol <= 0: run
 * exactly `iters` sweeps, no residual).  The loop, residual and stop flag stay on device.
 *   marginals: host array of l device pointers to mu_q (context dtype, >= 0, sum > 0; the
 *              library does not renormalise);
 *   u: host array of l device pointers, in = initial scalings, out = final (repr per opts);
 *   rep: host pointer, may be NULL.  Synchronises the context stream once at the end. */
MMOT_API mmot_status mmot_sinkhorn(mmot_ctx *ctx, const void *const *marginals, int iters, double tol,
                          void *const *u, mmot_report *rep);

/* Same as mmot_sinkhorn with HOST buffers: marginals_host[q] (context dtype) and u_host[q]
 * (float64, repr per opts) are copied to device staging buffers owned by the context, the
 * solve runs, u is copied back.  Pinned host memory gives asynchronous copies.
 * Synchronises once at the end. */
MMOT_API mmot_status mmot_sinkhorn_host(mmot_ctx *ctx, const void *const *marginals_host, int iters,
                               double tol, void *const *u_host, mmot_report *rep);

/* W = sum_i c(i) t(i), the linear transport cost of the plan t = K . (phi_1 x .. x phi_l)
 * (P:1037-1040), with a single factor h (Algorithm 4's return line P:652 applies h twice,
 * DESIGN.md A8).  Computed as h <phi_l, hatJ_l> with hatJ = sum E lambda^E prod phi carried
 * as the tangent of the same scans.  W: host pointer.  Synchronises. */
MMOT_API mmot_status mmot_cost(mmot_ctx *ctx, const void *const *u, double *W);

/* mmot_cost of the scalings the last mmot_sinkhorn_host left in the context's device staging
 * buffers (the host-buffer counterpart of mmot_cost: no further host<->device copy of u).
 * MMOT_EINVAL before the first mmot_sinkhorn_host of the context.  W: host pointer ([batch] for
 * batched contexts).  Synchronises. */
MMOT_API mmot_status mmot_cost_staged(mmot_ctx *ctx, double *W);

/* u_q <- the paper's initial scalings phi_q = 1/N: log phi = -log N (MMOT_LOG)
 * or 1/N (MMOT_LINEAR).  u: host array of l device pointers.  Asynchronous. */
MMOT_API mmot_status mmot_init_uniform(mmot_ctx *ctx, void *const *u);

/* Release all workspace.  NULL is a no-op. */
MMOT_API void mmot_destroy(mmot_ctx *ctx);

/* Static description of a status code. */
MMOT_API const char *mmot_strerror(mmot_status s);

/* Last detailed error message of the context ("" if none).  ctx may be NULL (global). */
MMOT_API const char *mmot_last_error(const mmot_ctx *ctx);

/* Library version as (major << 16 | minor). */
MMOT_API int mmot_version(void);

/* Launch plan of a context: grid points per chain P, number of chains, kernel family actually
 * used (MMOT_KERNEL_* value; 5 = 2-D grid, with chain_len = N1 and nchains = N2; 6 = the l = 6
 * lane-state family, one warp per 32-point chain with the 32 subset states on its lanes, which
 * AUTO l = 6 contexts use for updates, marginals and residuals (MMOT_KERNEL_TWO_WALK or MMOT_NO_LANES=1: the
 * two-walk kernels); chain_len / nchains then describe the two-walk layout the cost uses).  Any
 * output pointer may be NULL. */
MMOT_API mmot_status mmot_info(const mmot_ctx *ctx, int64_t *chain_len, int64_t *nchains, int *kernel);

/* Kernel-launch counter: number of CUDA kernels this context has launched so far. */
MMOT_API int64_t mmot_launch_count(const mmot_ctx *ctx);

/* Single-walk precision guard.  The single-walk family walks suffix states forward
 * through the subtractive inverse step; every product checks each chain's walked end state against
 * the exact suffix carry of the next chain (componentwise relative error <= 1e-11, which bounds the
 * error of every interior state).  If a check fails (scalings with large jumps, e.g. spanning
 * 1e+-50 between neighbouring points), mmot_sinkhorn / mmot_marginal / mmot_cost redo the call on a
 * two-walk context of the same problem before writing any output (single-walk mmot_marginal
 * therefore synchronises the stream once), and sharded contexts return MMOT_EPRECISION on every
 * rank.  Returns how many calls of this context were redone. */
MMOT_API int64_t mmot_fallback_count(const mmot_ctx *ctx);

/* Range fallback (a8).  When a product of the plain fp64 families leaves the fp64 range
 * (MMOT_EOVERFLOW: e.g. disjoint supports at small eta, where J_k spans e^-8000 .. e^+4000),
 * mmot_sinkhorn / mmot_marginal / mmot_cost of single-instance contexts redo the call from its
 * inputs on the stabilised family (MMOT_KERNEL_STABLE), and batched contexts redo exactly the failed
 * instances; uniform grids, not sharded (sharded contexts still return MMOT_EOVERFLOW on every rank).
 * Marginal / cost calls of a batched context that needed it run on the stabilised family from then
 * on.  MMOT_NO_STABLE=1 disables it.  Returns how many calls were redone. */
MMOT_API int64_t mmot_stable_fallback_count(const mmot_ctx *ctx);

/* All-marginals residual.  The residual check of mmot_sinkhorn (sum over k < l-1 of
 * ||phi_k J_k - mu_k||_1, Algorithm 1 line 7, generalised) needs every J_k on the same
 * end-of-sweep vectors.  Two-walk contexts with l <= 5 (uniform grid, one process) evaluate them in
 * ONE pass of the subset recurrence over all l scalings (2^l states: the states without marginal k
 * are exactly update k's states, so each J_k is a combine over the subsets without k) instead of
 * l-1 products, in a workspace of its own, so the update sequence keeps its fused operators.  Other
 * families keep the l-1 residual products (the persistent kernel folds the k = 0 term into the next
 * sweep).  MMOT_NO_ALLRES=1 disables it.  Returns how many checks used the single pass. */
MMOT_API int64_t mmot_allres_checks(const mmot_ctx *ctx);

/* Device-resident driver.  Single-process contexts run the sweep loop of mmot_sinkhorn as
 * ONE launch of a cached CUDA graph whose conditional WHILE node repeats a captured period of
 * sweeps (tol > 0: check_every sweeps ending with the residual check and the device stop rule;
 * tol <= 0: the periodic steady state after the first sweep(s)) until the sweeps are done or the
 * device stop flag is set -- no host round trip per sweep.  The persistent family runs a whole solve
 * in one kernel; sharded contexts and profiled contexts (mmot_profile_enable) keep host-issued
 * launches (MMOT_NO_GRAPH=1 forces them).  The graph is rebuilt when the vectors passed change.
 * Returns how many solves of this context used the graph. */
MMOT_API int64_t mmot_graph_solves(const mmot_ctx *ctx);

/* Pair family (batched contexts).  A batched Sinkhorn with a fixed sweep count (tol <= 0), a
 * uniform grid and a batch of at least MMOT_PAIR_MIN instances (default 4096) runs on two threads
 * per instance with no chain operators: each half of the grid is walked from its open end (where
 * the carry is the empty-set state), the halves' end states are swapped, and each half then walks
 * the other direction with the combine.  Scalings are stored as mantissas with one
 * exponent per 8 grid points (fp64 mantissas; fp32 mantissas and marginals in MMOT_F32 contexts).
 * MMOT_NO_PAIR=1 keeps the one-warp-per-instance kernel.  Returns how many solves of this context
 * used the pair family. */
MMOT_API int64_t mmot_pair_solves(const mmot_ctx *ctx);

/* Of those, the solves that also COMPUTED in fp32 (MMOT_F32 contexts, unless MMOT_PAIR_F64=1 is set
 * in the environment): the walks and combine in fp32 arithmetic with the states kept relative to the
 * 8-point slab exponents (linear fp32 values with a per-block integer exponent;
 * north_star's fp32 tolerance 1e-4), the division in fp64.  Instances whose states leave the fp32
 * range are redone in fp64 (mmot_pair_redo_count).  fp64 contexts compute in fp64. */
MMOT_API int64_t mmot_pair_f32_solves(const mmot_ctx *ctx);

/* Instances of fp32 pair solves whose states left the fp32 range and were redone in fp64 on a
 * batched context of their own (the one-warp-per-instance kernel), from the same inputs. */
MMOT_API int64_t mmot_pair_redo_count(const mmot_ctx *ctx);

/* CTA family (batched contexts, and the single-instance contexts mmot_create gives small problems).
 * A batched Sinkhorn whose batch fits one wave (<= the SM count) with l <= 4, N <= 4096, a uniform
 * grid and every instance inside (l-1)(x_max - x_min)/eta <= 500 runs one thread block per instance:
 * 256 chains, warp-level operator scans, all sweeps and residual checks in one launch (DESIGN.md
 * §5).  Scalings are plain fp64; a product that leaves the range reports EOVERFLOW and the instance
 * is redone on the stabilised family.  MMOT_NO_CTA=1 keeps the one-warp-per-instance kernel.
 * Returns how many solves of this context used the CTA family. */
MMOT_API int64_t mmot_cta_solves(const mmot_ctx *ctx);

/* Benchmark instrumentation.  While enabled, every tensor-vector product records CUDA events
 * on the context stream around its phases.  mmot_profile_read synchronises the stream and
 * returns, accumulated since the last read, the device milliseconds and product counts of
 *   ms[0] operator phase, ms[1] scan phase, ms[2] apply phase, ms[3] whole product,
 * and per mode in ms_mode[0..3] (marginal, update, residual, cost) with counts n_mode[0..3].
 * Either output pointer may be NULL. */
MMOT_API mmot_status mmot_profile_enable(mmot_ctx *ctx, int enable);
MMOT_API mmot_status mmot_profile_read(mmot_ctx *ctx, double *ms /*[4]*/, double *ms_mode /*[4]*/,
                                       int64_t *n_mode /*[4]*/);

#ifdef __cplusplus
}
#endif
#endif /* MMOT_H_ */
