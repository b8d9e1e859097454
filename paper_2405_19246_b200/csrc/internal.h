// internal.h -- host-side plan of one tensor-vector product and the kernel launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dp.cuh"

namespace mmot {

enum Mode : int {
    MODE_MARG = 0,  // out = phi_k * J_k                         (mmot_marginal)
    MODE_UPD = 1,   // phi_k = mu_k / J_k                        (Sinkhorn update)
    MODE_RES = 2,   // partial[c] = sum |phi_k J_k - mu_k|       (residual)
    MODE_COST = 3,  // partial[c] = sum phi_k * hatJ_k (duals)   (W)
    MODE_ALLRES = 4,  // NEXT-1: ONE pass of the 2^l-state DP over ALL l scalings (NB = l) gives every
                      // J_k (combine over the subsets without k); partial[c] = sum_{k<l-1} |phi_k J_k - mu_k|
};

constexpr int kGroup = 32;  // operators per group of the hierarchical scan when NB <= 3 (one warp)
// NB >= 4 composes a group sequentially in one thread (an op_compose of 2^NB-state operators is
// heavy): smaller groups shorten that serial chain at the price of more levels.
__host__ __device__ constexpr int group_of(int NB) { return NB <= 3 ? 32 : 8; }
constexpr double kSwGuardTol = 1e-11;  // single-walk guard: max relative error of a walked end state
constexpr double kSwBound = 1.0;   // max P * max_a a(l-a) * h/eta for the single-walk kernels      // operators composed per thread in the hierarchical scan
constexpr int kMaxLevels = 8;

// Sub-block length Q (registers hold Q suffix states) and max sub-blocks per chunk
// (local-memory checkpoints) for NB = l-1 bound marginals.
__host__ __device__ constexpr int sub_q(int NB) { return NB <= 2 ? 8 : (NB == 3 ? 4 : (NB == 4 ? 2 : 1)); }
__host__ __device__ constexpr int nsub_max(int NB) { return 256 >> NB; }
__host__ __device__ constexpr int chunk_max(int NB) { return sub_q(NB) * nsub_max(NB); }
__host__ __device__ constexpr int slab_s(int NB) { return NB <= 2 ? 16 : 8; }

// Lane-state family (lanes.cu, l = 6): chains of 32 points, warp per chain, lane = subset state.
constexpr int kLsB = 16;             // items per block of the lane-state operator scan (one warp each)
constexpr int kLsMaxLv = 7;          // scan levels: 16^7 chains
struct LsWork {
    int64_t P, C;                    // chain length (32), chains
    double *ops_f, *ops_b;           // [C][192] chain operators (chain order)
    int nlev;                        // scan levels (level 0 = chains)
    int64_t lv_n[kLsMaxLv];          // items per level
    double *lv_excl[kLsMaxLv][2];    // [n][192] exclusive in-block prefix per item, per direction
    double *lv_agg[kLsMaxLv][2];     // [n/16][192] block aggregates (= items of the next level)
    double *lv_car[kLsMaxLv][2];     // [n][32] state entering each item (scan order)
};

struct Plan {
    int NB;                          // l - 1
    int64_t N, P, nchunks;
    const double *bound[kMaxL];      // the NB bound scaling vectors, increasing marginal index
    const double *phik;              // phi_k (marg / res / cost)
    const double *muk;               // mu_k (upd / res)
    const double *mus[kMaxL];        // MODE_ALLRES: mu_0 .. mu_{l-2} (bound[] = all l scalings, NB = l)
    double *outk;                    // out (marg) or phi_k (upd); may alias phik for upd
    Weights W;
    int nlev;
    int64_t nlev_n[kMaxLevels];      // entries per level (level 0 = chunks)
    void *ops_f[kMaxLevels], *ops_b[kMaxLevels];
    void *car_f[kMaxLevels], *car_b[kMaxLevels];
    void *car_bi;                    // level 0: suffix state at the START of every chain (inclusive)
    int sw;                          // 1: single-walk kernels (stable regime, see mmot_create); vectors are
                                     //    then in the chain-blocked layout ((c/32)*32P + t*32 + c%32)
    int64_t nchp;                    // chain count rounded up to 32 (transposed row length)
    // sharded contexts (mmot_create_sharded): after the up-sweep the whole-shard operators are
    // written to agg_send ([2][SZ]: prefix, suffix), exch() all-gathers them into agg_all
    // ([world][2][SZ]) on the stream, and the carries entering the shard go to rank_car ([2][M])
    // restricted next-update scan (single-walk Sinkhorn, not sharded): nxr = 1 makes the update
    // kernel write the affine elements of the next update (rxe_*[0]) and the old parts of the next
    // carries (ncar_f, ncar_bi); rx_scan = 1 replaces the operator phase + full scan by the affine
    // scan, which writes the new parts of car_f[0] / car_bi
    int nxr, rx_scan;
    void *rxe_f[kMaxLevels], *rxe_b[kMaxLevels];    // affine elements per level
    void *rcar_f[kMaxLevels], *rcar_b[kMaxLevels];  // new-part carries per level (levels >= 1)
    void *ncar_f, *ncar_bi;                         // next update's full carries (old parts)
    void (*exch)(void *ctx, size_t doubles_per_rank, cudaStream_t s);
    void *exch_ctx;
    void *agg_send, *agg_all, *rank_car;
    int world, rank;
    double *partial;                 // nchunks partial sums
    int *stop;                       // device flag: nonzero -> every kernel returns at once
    int *status;                     // device status (mmot_status) of the run
    int *fail_iter;                  // device: sweep index of the first failure
    int iter;                        // current sweep index (for fail_iter) outside a solve
    const int *sweep = nullptr;      // inside a solve: device count of completed sweeps (fail_iter)
    // single-walk precision guard: every chain stores its walked end state (sw_end, [nchunks][M] in
    // T units) and k_sw_guard compares it with the exact inclusive suffix carry of the next chain;
    // a componentwise relative difference above kSwGuardTol sets *guard
    void *sw_end = nullptr;
    int *guard = nullptr;
    const LsWork *ls = nullptr;      // l = 6: the lane-state family's workspace (null: two-walk kernels)
    const double *lam = nullptr;     // non-uniform grid: per-edge decays [nchunks P + 1] (null: uniform)
    const double *hx = nullptr;      // non-uniform grid: edge lengths (cost duals)
};

// Enqueue one product (ops -> scan -> apply) of `mode` on `s`.  Returns the number of
// kernels launched through *launches (accumulated).
// with_ops = false skips the operator phase (operators already in ops_f/ops_b level 0, e.g.
// written by the previous fused update); next = true (MODE_UPD) fuses the operators of the
// NEXT update's bound set into the apply walk (cyclic bound order, see make_plan).
cudaError_t launch_product(const Plan &p, int mode, cudaStream_t s, int64_t *launches,
                           cudaEvent_t *ev = nullptr /* 4 events: before ops, after ops, after scan, after apply */,
                           bool with_ops = true, bool next = false);

// Lane-state family (l = 6): ops -> two-level scan -> apply, modes UPD / MARG / RES.
cudaError_t launch_ls_product(const Plan &p, const LsWork &w, int mode, cudaStream_t s, int64_t *launches);
cudaError_t ls_init_tables();  // composition term table on the current device (once; not capturable)

// Resident CTAs (of kWarpsPerCta warps) per SM of the single-walk update kernel.
int sw_blocks_per_sm(int NB);
constexpr int kWarpsPerCtaHost = 4;

// Deterministic single-block sum of partial[0..n) -> *out = scale * sum (+ *out if accumulate).
cudaError_t launch_sum(const double *partial, int64_t n, double *out, double scale, int accumulate,
                       const int *stop, cudaStream_t s, int64_t *launches);

// Natural <-> chain-blocked layout (x = c*P + t <-> (c/32)*32P + t*32 + c%32); op 0 copy, 1 exp, 2 log.
// flags != nullptr fuses launch_check into the pass (flags bit0 non-finite, bit1 negative; mass += sum
// when mass != nullptr).
cudaError_t launch_to_t(const double *src, double *dst, int64_t N, int64_t P, int64_t nchains, int64_t nchp, int op,
                        cudaStream_t s, int64_t *launches, int *flags = nullptr, double *mass = nullptr,
                        int allow_neg_inf = 0);
cudaError_t launch_from_t(const double *src, double *dst, int64_t N, int64_t P, int64_t nchains, int64_t nchp, int op,
                          cudaStream_t s, int64_t *launches);
constexpr int kSwSlab = 8;  // chain length of single-walk contexts is a multiple of this

// Batched contexts (batched.cu): one warp per instance, persistent over the sweeps.
struct BatchArgs {
    int l;
    int64_t N, batch;
    int P;                       // chain length (multiple of 8), 32 chains per instance
    double h;
    const double *eta;           // device [batch]
    double *phit[kMaxL];         // device [batch][N] mantissas of phi_q
    int *E;                      // device [batch][l][32] chain exponents
    const double *mu[kMaxL];     // device [batch][N]
    double *ops, *ckpt;          // scratch, sized by bat_scratch_bytes
    double *rsave = nullptr;     // [slots][N] scratch for the deferred residual (persistent kernel)
    const double *lam = nullptr; // non-uniform grids: [batch][ne] per-edge decays (null: uniform)
    const double *hx = nullptr;  // non-uniform grids: [ne] edge lengths
    int64_t ne = 0;              // edges per row: 32 P + 1
    int64_t slots;               // resident warps (= scratch slots)
    int iters, k;
    double *out;                 // [batch][N] (marginal)
    double *wout;                // [batch] (cost)
    int *status, *fail_iter;     // [batch]
    double tol;                  // residual tolerance (<= 0: run exactly iters sweeps)
    int check_every;             // residual cadence in sweeps
    int *iters_done, *converged; // [batch]
    double *resid;               // [batch] last residual (NaN if never computed)
};
int64_t bat_slots(int l);
// lam[b][e] = exp(-hx[e] / eta[b]) (1 where hx[e] = 0)
cudaError_t launch_bat_lambda(double *lam, const double *hx, const double *eta, int64_t batch, int64_t ne, cudaStream_t s);
// mass <- min over instances of sum_x mu[inst][x] (per-instance zero-mass check)
cudaError_t launch_bat_min_mass(const double *mu, int64_t batch, int64_t N, double *mass, cudaStream_t s,
                                int64_t *launches);
// what: 0 Sinkhorn (iters sweeps), 1 marginal k -> out, 2 cost -> wout
cudaError_t launch_batched(const BatchArgs &a, int what, cudaStream_t s, int64_t *launches);
// u: DEVICE array of l device pointers; import: u -> (phit, E), else (phit, E) -> u
cudaError_t launch_bat_convert(const BatchArgs &a, void *const *u_dev_ptrs, int import, int is_log, cudaStream_t s,
                               int64_t *launches);

// Pair family (pair.cu): large batches, two threads per instance (halves A = [0, nA), B mirrored),
// no chain operators; scalings as mantissas + one exponent per 8 positions.
struct PairPlan {
    int l;
    int64_t batch, N;
    int nA, nB;        // positions of the left half (ceil(N/2)) and of the mirrored right half
    int nslab;         // slabs of 8 positions per half: ceil(nA / 8)
    int64_t nblk;      // blocks of 16 instances (one warp each)
    double h;
    const double *eta; // [batch]
    void *phit;        // [l][nblk][nslab * 8][32] mantissas (double, or float if f32)
    void *mu;          // [l][nblk][nslab * 8][32] marginals (double, or float if f32)
    int *E;            // [nblk][nslab][l][2][32] exponent records: slab exponents E and the state
                       // scales G of the fp32 walks (decay envelope of E), pair.cu pr_xrec
    double *ckpt;      // [slots][nslab][2^(l-1)][32] (own state before each slab)
    int64_t slots;     // resident warps (checkpoint slots)
    int iters;
    int f32;           // fp32 storage of mantissas and marginals (MMOT_F32 contexts)
    int f32c;          // fp32 arithmetic as well (MMOT_F32 contexts unless MMOT_PAIR_F64 is set)
    int *status, *fail_iter, *iters_done, *converged;  // [batch]
    double *resid;     // [batch]
};
int64_t pair_slots();

// CTA family (cta.cu): one thread block per small instance (l <= 4, N <= 4096), 256 chains,
// warp-level operator scans; plain fp64 scalings (instances inside kCtaRange).
constexpr double kCtaRange = 500.0;  // max (l-1) (x_max - x_min) / eta of an instance
struct CtaPlan {
    int l;
    int64_t N, batch;
    int P;                          // chain length: cta_chain_len(N)
    double h;
    const double *eta;              // [batch]
    double *phi[kMaxL];             // [batch][N] linear scalings
    const double *mu[kMaxL];        // [batch][N]
    double *scr;                    // [batch][N] deferred-residual update of phi_0
    int iters, check_every;
    double tol;
    int *status, *fail_iter, *iters_done, *converged;  // [batch]
    double *resid;                  // [batch]
};
int cta_chain_len(int64_t N);
cudaError_t launch_cta_sinkhorn(const CtaPlan &cp, cudaStream_t s, int64_t *launches);
// op 0: u -> phi, 1: phi -> u (u_dev: DEVICE array of l device pointers)
cudaError_t launch_cta_convert(const CtaPlan &cp, void *const *u_dev, int op, int log_repr, cudaStream_t s,
                               int64_t *launches);
cudaError_t launch_pair_sinkhorn(const PairPlan &pp, cudaStream_t s, int64_t *launches);
// op 0: u -> mantissas + exponents; 1: -> u; 2: mu (fp64 [batch][N]) -> the pair layout.
// u_dev: DEVICE array of l device pointers.
cudaError_t launch_pair_convert(const PairPlan &pp, void *const *u_dev, int op, int log_repr, cudaStream_t s,
                                int64_t *launches);

// Allow `bytes` of dynamic shared memory for kernel `func` on the CURRENT device.  The attribute is
// per device, so it is set once per (kernel, device, size) (thread-safe cache).
void smem_attr(const void *func, size_t bytes);

// In-process collectives of virtual shard groups (several sharded contexts on one device, each
// driven by its own host thread and stream): out[i] = op_r src[r][i], op 0 = sum (double),
// op 1 = max (int).
constexpr int kMaxWorld = 16;
struct VPtrs {
    const void *p[kMaxWorld];
};
cudaError_t launch_vreduce(const VPtrs &src, int world, int n, int op, void *out, cudaStream_t s, int64_t *launches);

// Stabilised family (stable.cu): log-domain subset recurrence, one warp per instance.  The only
// family for l = 7, 8 (2^(l-1) = 64 / 128 subset states: 2 / 4 per lane).
constexpr int kStMaxL = 8;
struct SPlan {
    int l;
    int64_t N, batch;
    double h;                    // grid spacing
    const double *eta;           // device [batch]
    double *g[kStMaxL];          // device [batch][N] log scalings (in/out)
    const double *mu[kStMaxL];   // device [batch][N] marginals (linear)
    double *scratch;             // device [slots][scratch_per_warp]
    int64_t scratch_per_warp;    // 2 N 2^(l-1) doubles
    int64_t slots;               // resident warps (scratch slots)
    const int *sel;              // device [batch] 1 = process (null: all instances)
    int iters, check_every, k;
    double tol;
    double *out, *wout;          // marginal [batch][N] / cost [batch]
    double hc;                   // cost factor h
    int *status, *fail_iter, *iters_done, *converged;  // device [batch]
    double *resid;               // device [batch]
};
// what: 0 Sinkhorn (iters sweeps), 1 marginal k -> out, 2 cost -> wout
cudaError_t launch_stable(const SPlan &sp, int what, cudaStream_t s, int64_t *launches);
// in -> out for the selected instances: op 0 copy, 1 log, 2 exp
cudaError_t launch_st_convert(const double *in, double *out, int64_t batch, int64_t N, const int *sel, int op,
                              cudaStream_t s, int64_t *launches);

// 2-D grids (grid2d.cu, §4.1): l = 3 on an N x M mesh, column-major vectors x[i1 + N i2].
struct G2Plan {
    int64_t N, M;                // rows (inner dimension, lambda1), columns (outer, lambda2)
    Weights Wi;                  // inner weights w_a = lambda1^{a(3-a)} and e_a (cost tangent)
    double wo1, wo2;             // outer weights lambda2^{1*2}, lambda2^{2*1}
    const double *a, *b;         // the two bound scalings
    const double *phik, *muk;    // free marginal's scaling / target (per mode)
    double *outk;                // marginal output or the new phi_k
    double *Fa, *Fb, *Ga, *Gb;   // [N M] column recursions
    void *Y;                     // [6][M][N] inner products (T)
    void *st;                    // [6 M][N][3] inner suffix states (T)
    void *Gab;                   // [M + 1][N] output-space suffix states (T)
    double *partial;             // [N] per-row partial sums (residual / cost)
    int *status, *stop, *fail_iter;
    int iter;
};
cudaError_t launch_g2_product(const G2Plan &p, int mode, cudaStream_t s, int64_t *launches);
cudaError_t launch_g2_transpose(const double *in, double *out, int64_t N, int64_t M, cudaStream_t s,
                                int64_t *launches);

// Elementwise helpers.
// fp32 <-> fp64 (to_f64: float in -> double out, else double in -> float out)
cudaError_t launch_convert(const void *in, void *out, int64_t n, int to_f64, cudaStream_t s, int64_t *launches);
cudaError_t launch_exp(const double *in, double *out, int64_t n, cudaStream_t s, int64_t *launches);
cudaError_t launch_log(const double *in, double *out, int64_t n, cudaStream_t s, int64_t *launches);
cudaError_t launch_fill(double *out, double v, int64_t n, cudaStream_t s, int64_t *launches);
// Validate marginals / scalings.  flags: bit0 non-finite, bit1 negative; mass[q] += sum.
cudaError_t launch_check(const double *v, int64_t n, int allow_neg_inf, int *flags, double *mass,
                         cudaStream_t s, int64_t *launches);
// After checks: turn flags/mass into a status and stop flag.
cudaError_t launch_check_finish(const int *flags, const double *mass, int nvec, int nmarg, int *status,
                                int *stop, int *fail_iter, cudaStream_t s, int64_t *launches);
// End of a residual evaluation: res = *acc; iters_done = *sweep; if res <= tol stop (converged).
cudaError_t launch_resid_finish(double *acc, double tol, const int *sweep, double *res_out, int *iters_done,
                                int *converged, int *stop, cudaStream_t s, int64_t *launches);
// End of a sweep: unless stopped, ++*sweep and iters_done = *sweep.
cudaError_t launch_sweep_done(int *sweep, int *iters_done, const int *stop, cudaStream_t s, int64_t *launches);
// Device-resident loop: ++*done; conditional h = (*done < *n && !*stop) (graph WHILE node body end).
cudaError_t launch_loop_cond(cudaGraphConditionalHandle h, int *done, const int *n, const int *stop, cudaStream_t s,
                             int64_t *launches);

}  // namespace mmot
