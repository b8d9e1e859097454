// batched.cu -- many independent MMOT instances (BASELINE C5: 8192 x (l=5, N=4096), per-instance
// eta), one warp per instance, persistent over the Sinkhorn sweeps (north_star (b)).
//
// Per instance the grid is cut into 32 chains (lane r <-> points [rP, (r+1)P)), and every
// quantity is kept in the scale of its chain: the scalings are stored as
//     phi_q[x] = phit_q[x] * 2^{E_q[r]}          (fp64 mantissa field, one integer exponent per
//                                                   chain and marginal, max phit in [1, 2))
// because at eta = 1e-3 |log phi| reaches ~1.8e3, beyond fp64's range.  A state
// F[S] of a chain is stored relative to 2^{sum_{q in S} E_q[r]}; conjugating a chain operator by
// such a per-marginal diagonal scaling keeps its shift-invariant form (entries G_c[V] pick up
// 2^{-sum_{q in V} E_q}), so every walk runs on the chain's own mantissas unchanged.  Carries
// cross a chain boundary through the exact power-of-two conversion
//     F~_{r+1}[S] = F~_r[S] * 2^{sum_{q in S} (E_q[r] - E_q[r+1])}
// and are propagated lane to lane inside the warp (31 sequential operator applications per
// direction, each between neighbouring chains only, so no intermediate leaves the fp64 range).
//
// One Sinkhorn update phi_k <- mu_k / J_k of an instance:
//   1. prefix / suffix carry propagation with the chain operators of this update's bound set;
//   2. walk 1 (right to left): suffix states, checkpoint at every slab end (global scratch);
//   3. walk 2 (left to right): prefix states, suffix states rebuilt per half-slab from the
//      checkpoint, combine J_k[m] = sum_S F_m[S] w_{|S|+1} B_{m+1}[S^c], phi_k = mu_k / J_k;
//   4. renormalise the chain exponent of phi_k (max mantissa in [1, 2));
//   5. chain operators (extended walk, prefix/suffix duality) of the next update's bound set.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "internal.h"
#include "walk.cuh"

namespace mmot {

constexpr int kBS = 8;          // slab = checkpoint block (points per chain)
constexpr int kBWarps = 8;      // warps (instances) per CTA (one CTA per SM, all in lockstep)
constexpr int kRenorm = 96;     // lazy renormalisation threshold: |max exponent of a chain| (products of l <= 5 mantissas stay below 2^480)
static const int g_renorm = [] { const char *e = getenv("MMOT_BAT_RENORM"); return e ? atoi(e) : kRenorm; }();

// exact 2^n as a double (0 below the normal range, inf above)
__device__ __forceinline__ double pow2i(int n) {
    if (n < -1022) return 0.0;
    if (n > 1023) return __longlong_as_double(0x7ff0000000000000ll);
    return __longlong_as_double((long long)(n + 1023) << 52);
}
// x * 2^n without forming an out-of-range factor
__device__ __forceinline__ double scale2(double x, int n) {
    if (n >= -1022 && n <= 1023) return x * pow2i(n);
    const int h = n / 2;
    return (x * pow2i(h)) * pow2i(n - h);
}
// 2^n with n clamped to the normal range (branch-free)
__device__ __forceinline__ double pow2c(int n) {
    n = max(-1022, min(1023, n));
    return __longlong_as_double((long long)(n + 1023) << 52);
}
// floor(log2 x) of a positive normal double; very negative for 0 / denormals
__device__ __forceinline__ int ilog2d(double x) {
    const int e = (int)((__double_as_longlong(x) >> 52) & 0x7ff);
    return e == 0 ? -1000000 : e - 1023;
}

template <int NB>
__device__ __forceinline__ void bweights(double (&wt)[NB + 2], double eta, double h) {
    constexpr int L = NB + 1;
#pragma unroll
    for (int a = 0; a <= NB + 1; ++a) wt[a] = a <= L ? exp(-(double)(a * (L - a)) * h / eta) : 0.0;
}

// Scale state vector v (relative to chain scale) by 2^{sum_{b in S} d[b]} for every S.
template <int NB, typename T>
__device__ __forceinline__ void vec_shift(T (&v)[1 << NB], const int (&d)[NB > 0 ? NB : 1]) {
#pragma unroll
    for (int S = 1; S < (1 << NB); ++S) {
        int n = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
            if ((S >> b) & 1) n += d[b];
        // branch-free exact 2^n in two factors (|n| up to ~2000 without forming 0 / inf early)
        const int h1 = n >> 1;
        const double a1 = pow2c(h1), a2 = pow2c(n - h1);
        if constexpr (sizeof(T) == sizeof(double)) {
            v[S] = (v[S] * a1) * a2;
        } else {
            reinterpret_cast<Dual &>(v[S]).v = (reinterpret_cast<Dual &>(v[S]).v * a1) * a2;
            reinterpret_cast<Dual &>(v[S]).d = (reinterpret_cast<Dual &>(v[S]).d * a1) * a2;
        }
    }
}

struct BPlan {
    int l;
    int64_t N, batch;
    int P;                          // chain length (multiple of kBS), 32 chains per instance
    double h;
    const double *eta;              // [batch]
    double *phit[kMaxL];            // [batch][N] mantissas
    int *E;                         // [batch][l][32] chain exponents
    const double *mu[kMaxL];        // [batch][N]
    double *ops;                    // scratch [slot][2][SZ][32]
    double *ckpt;                   // scratch [slot][P/kBS][M][32] (x2 for duals)
    const double *lam;              // non-uniform grids: [batch][ne] lambda_e = exp(-h_e / eta) (else null)
    const double *hx;               // non-uniform grids: [ne] edge lengths h_e (edge e between points e-1, e)
    int64_t ne;                     // 32 P + 1 (edges 0 .. 32 P; 1 / 0 outside 1 .. N-1)
    double hc;                      // cost factor: h (uniform: hatJ counts edges) or 1 (edge lengths in the tangent)
    double *rsave;                  // [slot][N]: phit_0 before the update that closes a deferred residual
    int64_t slots;                  // resident warps (scratch slots)
    int iters;
    int k;                          // product mode: free marginal
    double *out;                    // MARG: [batch][N]
    double *wout;                   // COST: [batch]
    int *status;                    // [batch] per-instance status (0 ok, EOVERFLOW)
    int *fail_iter;                 // [batch]
    int renorm;                     // lazy renormalisation threshold (kRenorm)
    double tol;                     // residual tolerance (<= 0: fixed sweeps)
    int check_every;                // residual cadence (sweeps)
    int *iters_done;                // [batch]
    int *converged;                 // [batch]
    double *resid;                  // [batch]
};

// Non-uniform grids (paper footnote P:182): weights of edge e of instance inst (walk.cuh).
template <int NB, typename T>
__device__ __forceinline__ void pweights(T (&w)[NB + 2], const BPlan &bp, int64_t inst, int64_t e) {
    pweights_val<NB, T>(w, __ldg(bp.lam + inst * bp.ne + e), sizeof(T) == sizeof(double) ? 0.0 : __ldg(bp.hx + e));
}


// ---------------------------------------------------------------------------------------
// Chain operator walk (extended operator, dp.cuh opx_*) of the bound set (k+1..k+NB mod l);
// stores prefix op (dir 0) and suffix op (dir 1) of every lane into its slot's scratch.
template <int NB, typename T, bool PTS>
__device__ void bat_ops(const BPlan &bp, int64_t inst, int k, const T (&wt)[NB + 2], double *buf, T *ops, int lane) {
    constexpr int M = 1 << NB;
    constexpr int S = kBS;
    constexpr int TILE = 32 * (S + 1);
    constexpr int SZ = OpShape<NB>::SZ;
    const int64_t N = bp.N;
    const double *vecs[NB > 0 ? NB : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b) vecs[b] = bp.phit[(k + 1 + b) % (NB + 1)] + inst * N;
    const int ns = bp.P / S;
    T G[NB + 1][M];
    opx_identity<NB, T>(G);
    double f[NB > 0 ? NB : 1];
    slab_issue<S, NB>(buf, vecs, 0, bp.P, N, 0, lane);
    cp_async_commit();
    for (int s = 0; s < ns; ++s) {
        if (s + 1 < ns) slab_issue<S, NB>(buf + ((s + 1) & 1) * NB * TILE, vecs, 0, bp.P, N, s + 1, lane);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const double *cur = buf + (s & 1) * NB * TILE;
#pragma unroll 1
        for (int j = 0; j < S; ++j) {
            slab_f<NB, S>(f, cur, lane, j);
            if constexpr (PTS) {
                T wx[NB + 2];
                pweights<NB, T>(wx, bp, inst, (int64_t)lane * bp.P + s * S + j);  // edge into the point
                opx_step<NB, T>(G, wx, f, s == 0 && j == 0);
            } else {
                opx_step<NB, T>(G, wt, f, s == 0 && j == 0);
            }
        }
        __syncwarp();
    }
    T pf[SZ], pb[SZ];
#pragma unroll
    for (int i = 0; i < SZ; ++i) pf[i] = pb[i] = zero_of(T{});
    if constexpr (PTS) {
        T win[NB + 2], wout[NB + 2];
        pweights<NB, T>(win, bp, inst, (int64_t)lane * bp.P);             // entry edge of the chain
        pweights<NB, T>(wout, bp, inst, (int64_t)(lane + 1) * bp.P);      // exit edge
        opx_store_pts<NB, T>(G, win, wout, pf, pb);
    } else {
        opx_store<NB, T>(G, wt, pf, pb);
    }
#pragma unroll
    for (int i = 0; i < SZ; ++i) {
        ops[(0 * SZ + i) * 32 + lane] = pf[i];
        ops[(1 * SZ + i) * 32 + lane] = pb[i];
    }
    __syncwarp();
}

// Carries of this update's bound set: Fin = prefix state entering the chain, Bend = suffix
// state at the chain end (both in the chain's scale).  E[q] = this lane's chain exponents.
template <int NB, typename T, bool FULLCH>
__device__ void bat_carries(const T *ops, int k, const int (&E)[kMaxL], T (&Fin)[1 << NB], T (&Bend)[1 << NB], int lane,
                            const BPlan &bp) {
    // FULLCH: all 32 chains hold grid points (constant trip counts, the common case)
    const int nch = FULLCH ? 32 : (int)((bp.N + bp.P - 1) / bp.P);
    // nch = chains holding grid points (lanes >= nch walk only points beyond N): the carries need
    // nch - 1 sequential steps per direction, not 31 (small N, C1)
    constexpr int M = 1 << NB;
    constexpr int SZ = OpShape<NB>::SZ;
    constexpr int L = NB + 1;
    int Eb[NB > 0 ? NB : 1], Enx[NB > 0 ? NB : 1], Epv[NB > 0 ? NB : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        int e = 0;
#pragma unroll
        for (int q = 0; q < L; ++q)
            if (q == (k + 1 + b) % L) e = E[q];
        Eb[b] = e;
        Enx[b] = __shfl_down_sync(0xffffffffu, e, 1);
        Epv[b] = __shfl_up_sync(0xffffffffu, e, 1);
    }
    T G[NB + 1][M];
    {
        T tmp[SZ];
#pragma unroll
        for (int i = 0; i < SZ; ++i) tmp[i] = ops[(0 * SZ + i) * 32 + lane];
        op_load<NB, T>(G, tmp);
    }
    // prefix: lane s applies its operator to the carry it received, converts to chain s+1's
    // scale, hands it on
    T cur[M], y[M];
    vec_unit<NB, T>(cur);
    vec_unit<NB, T>(Fin);
    int d[NB > 0 ? NB : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b) d[b] = Eb[b] - Enx[b];
#pragma unroll 1
    for (int s = 0; s < nch - 1; ++s) {
        op_apply<NB, T>(G, cur, y);
        vec_shift<NB, T>(y, d);
#pragma unroll
        for (int S = 0; S < M; ++S) {
            if constexpr (sizeof(T) == sizeof(double)) {
                cur[S] = __shfl_sync(0xffffffffu, y[S], s);
            } else {
                reinterpret_cast<Dual &>(cur[S]).v = __shfl_sync(0xffffffffu, reinterpret_cast<Dual &>(y[S]).v, s);
                reinterpret_cast<Dual &>(cur[S]).d = __shfl_sync(0xffffffffu, reinterpret_cast<Dual &>(y[S]).d, s);
            }
        }
        if (lane == s + 1) {
#pragma unroll
            for (int S = 0; S < M; ++S) Fin[S] = cur[S];
        }
    }
    {
        T tmp[SZ];
#pragma unroll
        for (int i = 0; i < SZ; ++i) tmp[i] = ops[(1 * SZ + i) * 32 + lane];
        op_load<NB, T>(G, tmp);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) d[b] = Eb[b] - Epv[b];
    vec_unit<NB, T>(cur);
    vec_unit<NB, T>(Bend);
#pragma unroll 1
    for (int s = nch - 1; s > 0; --s) {
        op_apply<NB, T>(G, cur, y);
        vec_shift<NB, T>(y, d);
#pragma unroll
        for (int S = 0; S < M; ++S) {
            if constexpr (sizeof(T) == sizeof(double)) {
                cur[S] = __shfl_sync(0xffffffffu, y[S], s);
            } else {
                reinterpret_cast<Dual &>(cur[S]).v = __shfl_sync(0xffffffffu, reinterpret_cast<Dual &>(y[S]).v, s);
                reinterpret_cast<Dual &>(cur[S]).d = __shfl_sync(0xffffffffu, reinterpret_cast<Dual &>(y[S]).d, s);
            }
        }
        if (lane == s - 1) {
#pragma unroll
            for (int S = 0; S < M; ++S) Bend[S] = cur[S];
        }
    }
}

// Walk 1 (right to left) from Bend: checkpoint B at every slab end x0 + (s+1) S, s = 0..ns-1
// (the last one is Bend itself).  ck layout [s][M][32].
template <int NB, typename T, bool PTS>
__device__ void bat_walk1(const BPlan &bp, int64_t inst, int k, const T (&wt)[NB + 2], T (&st)[1 << NB], double *buf,
                          T *ck, int lane) {
    constexpr int M = 1 << NB;
    constexpr int S = kBS;
    constexpr int TILE = 32 * (S + 1);
    const int64_t N = bp.N;
    const double *vecs[NB > 0 ? NB : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b) vecs[b] = bp.phit[(k + 1 + b) % (NB + 1)] + inst * N;
    const int ns = bp.P / S;
    double f[NB > 0 ? NB : 1];
    slab_issue<S, NB>(buf, vecs, 0, bp.P, N, ns - 1, lane);
    cp_async_commit();
    for (int t = 0; t < ns; ++t) {
        const int s = ns - 1 - t;
#pragma unroll
        for (int S2 = 0; S2 < M; ++S2) ck[(s * M + S2) * 32 + lane] = st[S2];
        if (s > 0) slab_issue<S, NB>(buf + ((t + 1) & 1) * NB * TILE, vecs, 0, bp.P, N, s - 1, lane);
        cp_async_commit();
        if (s == 0) break;
        cp_async_wait<1>();
        __syncwarp();
        const double *cur = buf + (t & 1) * NB * TILE;
#pragma unroll 1
        for (int jj = S - 1; jj >= 0; --jj) {
            slab_f<NB, S>(f, cur, lane, jj);
            if constexpr (PTS) {
                T wx[NB + 2];
                pweights<NB, T>(wx, bp, inst, (int64_t)lane * bp.P + s * S + jj + 1);  // edge to the right
                dp_diag<NB, T, true>(st, wx);
            } else {
                dp_diag<NB, T, true>(st, wt);
            }
            dp_place<NB, T>(st, f);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    __syncwarp();
}

// Walk 2 (left to right): prefix states from Fin, suffix states rebuilt per sub-block of Q
// points from the slab-end checkpoint, combine, and the mode's epilogue.
//   MODE_UPD : phit_k <- mu_k / J (provisional scale 2^{-sum_b E_b}), returns max exponent
//   MODE_MARG: out = phi_k J (true scale)
//   MODE_COST: acc += phi_k hatJ (true scale)
template <int NB, typename T, int MODE, int Q, bool PTS>
__device__ int bat_walk2(const BPlan &bp, int64_t inst, int k, const T (&wt)[NB + 2], T (&F)[1 << NB], double *buf,
                         const T *ck, int sumE_bound, int Ek, double &acc, bool &bad, int lane, bool res = false,
                         const double *oldv = nullptr, int e_old = 0) {
    constexpr int M = 1 << NB;
    constexpr int S = kBS;
    constexpr int TILE = 32 * (S + 1);
    constexpr int NV = NB + 1;     // bound vectors + (mu_k | phi_k)
    constexpr int QPS = S / Q;
    const int64_t N = bp.N;
    const double *vecs[NV];
#pragma unroll
    for (int b = 0; b < NB; ++b) vecs[b] = bp.phit[(k + 1 + b) % (NB + 1)] + inst * N;
    vecs[NB] = (MODE == MODE_UPD && !res) ? bp.mu[k] + inst * N : bp.phit[k] + inst * N;
    double *outv = MODE == MODE_UPD ? bp.phit[k] + inst * N : (MODE == MODE_MARG ? bp.out + inst * N : nullptr);
    const int ns = bp.P / S;
    const int64_t x0 = (int64_t)lane * bp.P;
    double f[NB > 0 ? NB : 1];
    double *obuf = buf + 2 * NV * TILE;
    int emax = -1000000;
    const int e_true = sumE_bound + Ek;  // exponent of phi_k J_k's chain scale (MARG / COST / residual)
    // residual products run through the UPD instantiation (one code copy): phi_k is read from the
    // stage slot that holds mu_k in updates, mu_k straight from global memory
    const bool shok = Ek >= -1022 && Ek <= 1022 && !res;
    const double shsc = MODE == MODE_UPD && shok ? pow2i(-Ek) : 1.0;  // UPD: Ek = pending shift of phi_k
    slab_issue<S, NV>(buf, vecs, 0, bp.P, N, 0, lane);
    cp_async_commit();
    for (int s = 0; s < ns; ++s) {
        if (s + 1 < ns) slab_issue<S, NV>(buf + ((s + 1) & 1) * NV * TILE, vecs, 0, bp.P, N, s + 1, lane);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const double *cur = buf + (s & 1) * NV * TILE;
        T bend[M];
#pragma unroll
        for (int S2 = 0; S2 < M; ++S2) bend[S2] = ck[(s * M + S2) * 32 + lane];
#pragma unroll 1
        for (int jb = 0; jb < QPS; ++jb) {
            T st[M];
#pragma unroll
            for (int S2 = 0; S2 < M; ++S2) st[S2] = bend[S2];
            // walk the sub-blocks right of this one back to its right end
#pragma unroll
            for (int i = S - 1; i >= (jb + 1) * Q; --i) {
                slab_f<NB, S>(f, cur, lane, i);
                if constexpr (PTS) {
                    T wx[NB + 2];
                    pweights<NB, T>(wx, bp, inst, x0 + (int64_t)s * S + i + 1);
                    dp_diag<NB, T, true>(st, wx);
                } else {
                    dp_diag<NB, T, true>(st, wt);
                }
                dp_place<NB, T>(st, f);
            }
            T H[Q][M];
#pragma unroll
            for (int i = Q - 1; i >= 0; --i) {
                if constexpr (PTS) {
                    T wx[NB + 2];
                    pweights<NB, T>(wx, bp, inst, x0 + (int64_t)s * S + jb * Q + i + 1);
                    dp_diag<NB, T, true>(st, wx);
                } else {
                    dp_diag<NB, T, true>(st, wt);
                }
#pragma unroll
                for (int S2 = 0; S2 < M; ++S2) H[i][S2] = st[S2];
                if (i > 0) {
                    slab_f<NB, S>(f, cur, lane, jb * Q + i);
                    dp_place<NB, T>(st, f);
                }
            }
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                const int jx = jb * Q + i;
                slab_f<NB, S>(f, cur, lane, jx);
                if constexpr (PTS) {
                    T wx[NB + 2];
                    pweights<NB, T>(wx, bp, inst, x0 + (int64_t)s * S + jx);
                    dp_diag<NB, T, true>(F, wx);
                } else {
                    dp_diag<NB, T, true>(F, wt);
                }
                dp_place<NB, T>(F, f);
                const T J = combine<NB, T>(F, H[i]);
                const double jv = value_of(J);
                const double vk = cur[(NB * 32 + lane) * (S + 1) + jx];  // mu_k (UPD) or phit_k
                if (MODE == MODE_UPD && res) {
                    // |m_k - mu_k| (P:168 generalised)
                    const int64_t x = x0 + (int64_t)s * S + jx;
                    if (x < N) acc += fabs(scale2(vk * jv, e_true) - __ldg(bp.mu[k] + inst * N + x));
                } else if (MODE == MODE_UPD) {
                    const double q = div_nr1(vk, jv);
                    const bool nz = nonzero(vk);
                    const int64_t x = x0 + (int64_t)s * S + jx;
                    // deferred residual term of the previous sweep: |phi_k(old) J_k - mu_k| (the
                    // bound vectors are that sweep's end-of-sweep vectors; a7, "free" k = 1 term)
                    if (oldv && x < N) acc += fabs(scale2(oldv[x] * jv, sumE_bound + e_old) - vk);  // rewritten in-kernel: no __ldg
                    bad |= nz && x < N && !finite_positive(q);
                    const double o = nz ? (shok ? q * shsc : scale2(q, -Ek)) : 0.0;
                    obuf[lane * (S + 1) + jx] = o;
                    if (nz) emax = max(emax, ilog2d(o));
                } else if (MODE == MODE_MARG) {
                    obuf[lane * (S + 1) + jx] = scale2(vk * jv, e_true);
                } else if (MODE == MODE_COST) {
                    if constexpr (sizeof(T) == sizeof(Dual)) acc += scale2(vk * reinterpret_cast<const Dual &>(J).d, e_true);
                }
            }
        }
        __syncwarp();
        if ((MODE == MODE_UPD && !res) || MODE == MODE_MARG) {
            slab_store<S>(obuf, outv, 0, 32, bp.P, N, s, lane);
            __syncwarp();
        }
    }
    return emax;
}

// phit_k *= 2^{-shift_r} on every chain r whose lane asked for it (shift 0 = untouched); the
// warp sweeps the instance's vector with coalesced accesses (lane i takes elements i, i+32, ...).
__device__ void bat_rescale(double *v, int64_t N, int P, int shift, int lane) {
    const bool any = __any_sync(0xffffffffu, shift != 0);
    if (!any) return;
    for (int64_t x0 = 0; x0 < N; x0 += 32 * 4) {
        double t[4];
        int sh[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t x = x0 + u * 32 + lane;
            sh[u] = __shfl_sync(0xffffffffu, shift, (int)(x / P < 31 ? x / P : 31));
            t[u] = (x < N && sh[u] != 0) ? v[x] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t x = x0 + u * 32 + lane;
            if (x < N && sh[u] != 0) v[x] = scale2(t[u], -sh[u]);
        }
    }
}

// ---------------------------------------------------------------------------------------
// Persistent Sinkhorn: each warp loops over instances; per instance `iters` sweeps of the l
// Gauss-Seidel updates, all on device.
template <int NB, bool PTS, bool CHK>
__global__ void __launch_bounds__(kBWarps * 32) k_bat_sinkhorn(BPlan bp) {
    // CHK = false (tol <= 0, e.g. C5): no residual slots at all -- the residual and deferral code
    // is compiled out, which keeps the walk registers of the fixed-sweep case unchanged
    // The warps of a CTA run the phases of an update in lockstep (CTA barriers between phases),
    // so only one phase's code is hot in the SM's instruction cache at a time: this kernel is
    // instruction-fetch bound otherwise (ncu: "no instruction" was the top stall).
    using T = double;
    constexpr int L = NB + 1;
    constexpr int M = 1 << NB;
    constexpr int S = kBS;
    constexpr int TILE = 32 * (S + 1);
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t slot = (int64_t)blockIdx.x * kBWarps + warp;
    double *buf = smem + (size_t)warp * (2 * L + 1) * TILE;
    T *ops = bp.ops + slot * 2 * OpShape<NB>::SZ * 32;
    T *ck = bp.ckpt + slot * (int64_t)(bp.P / S) * M * 32;
    for (int64_t base = (int64_t)blockIdx.x * kBWarps; base < bp.batch; base += bp.slots) {
        const int64_t inst = base + warp;
        const bool active = inst < bp.batch;
        T wt[NB + 2];
        bweights<NB>(wt, active ? bp.eta[inst] : 1.0, bp.h);
        int E[kMaxL];
#pragma unroll
        for (int q = 0; q < kMaxL; ++q) E[q] = (q < L && active) ? bp.E[(inst * L + q) * 32 + lane] : 0;
        int Sh[kMaxL];  // per marginal: E_q = -sum_{p != q} E_p + Sh_q (lazy renormalisation)
#pragma unroll
        for (int q = 0; q < kMaxL; ++q) {
            int s2 = 0;
#pragma unroll
            for (int p = 0; p < L; ++p) s2 += E[p];
            Sh[q] = q < L ? s2 : 0;
        }
        bool bad = false;
        int fail = -1;
        int done_it = 0;
        bool conv = false;
        double last_res = __longlong_as_double(0x7ff8000000000000ll);  // NaN: never computed
        if (active) bat_ops<NB, T, PTS>(bp, inst, 0, wt, buf, ops, lane);
        __syncthreads();
        // One sweep = l update slots and, on check sweeps, l-1 residual slots
        // (Res_t = sum_{k<l-1} ||phi_k J_k - mu_k||_1 on the end-of-sweep vectors, Algorithm 1
        // line 7, P:168 generalised; stop at the first Res <= tol).  Every slot runs the same
        // code (one copy of each phase: the kernel is register- and instruction-cache-bound); the
        // chain operators of the next slot's bound set are built at the end of each slot.
        // residual of a check sweep t < iters: the k = 0 term is taken inside sweep t+1's first update
        // (same bound vectors), the other l-2 terms in residual slots at the end of sweep t; if the
        // total meets tol, that first update is undone (phit_0 restored, exponents kept)
        bool pend = false;
        double pres = 0.0;
        int pt = 0;
        double *rsave = bp.rsave + slot * bp.N;
        for (int t = 1; t <= bp.iters; ++t) {
            const bool run = active && !conv && !__any_sync(0xffffffffu, bad);
            const bool check = CHK && bp.tol > 0 && (t % bp.check_every == 0 || t == bp.iters);
            const bool defer = check && t < bp.iters;
            const int nslots = L + (check ? (defer ? L - 2 : L - 1) : 0);
            const int roff = defer ? 1 : 0;  // residual slot sl -> k = sl - L + roff
            double res = 0.0;
            bool live = run;
            for (int sl = 0; sl < nslots; ++sl) {
                const bool upd = sl < L;
                const int k = upd ? sl : sl - L + roff;
                const bool close = upd && k == 0 && pend && live;  // this update closes sweep pt's residual
                T F[M], B[M];
                if (live) {
                    if (31 * (int64_t)bp.P < bp.N) bat_carries<NB, T, true>(ops, k, E, F, B, lane, bp);
                    else bat_carries<NB, T, false>(ops, k, E, F, B, lane, bp);
                }
                __syncthreads();
                if (live) bat_walk1<NB, T, PTS>(bp, inst, k, wt, B, buf, ck, lane);
                if (close) {
                    // keep phit_0 of sweep pt (coalesced copy) for the residual and a possible undo
                    const double *src = bp.phit[0] + inst * bp.N;
                    for (int64_t x = lane; x < bp.N; x += 32) rsave[x] = src[x];
                    __syncwarp();
                }
                __syncthreads();
                int sumE = 0, Ek = 0, shk = 0;
#pragma unroll
                for (int q = 0; q < L; ++q) {
                    if (q != k) sumE += E[q];
                    else {
                        Ek = E[q];
                        shk = Sh[q];
                    }
                }
                if (live) {
                    double acc = 0.0;
                    bool b2 = false;
                    // updates: phit_k is written as (mu_k / J~) * 2^{-sh_k}, sh_k = the shift chosen at
                    // the previous update of marginal k (lazy renormalisation: rescaled only when the
                    // chain's maximum exponent drifts beyond +-renorm)
                    const int emax = bat_walk2<NB, T, MODE_UPD, 4, PTS>(bp, inst, k, wt, F, buf, ck, sumE, upd ? shk : Ek,
                                                                        acc, b2, lane, !upd, close ? rsave : nullptr, Ek);
                    bool undone = false;
                    if (close) {
                        double tot = acc;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
                        tot += pres;
                        pend = false;
                        last_res = tot;
                        if (tot <= bp.tol) {
                            // converged at sweep pt: undo this update
                            double *dst = bp.phit[0] + inst * bp.N;
                            for (int64_t x = lane; x < bp.N; x += 32) dst[x] = rsave[x];
                            __syncwarp();
                            conv = true;
                            done_it = pt;
                            live = false;
                            undone = true;
                        }
                    }
                    if (upd && !undone) {
                        if (b2 && fail < 0) fail = t;
                        bad |= b2;
                        const int resc = (emax > -1000000 && (emax > bp.renorm || emax < -bp.renorm)) ? emax : 0;
                        // (walk 2 ended with a __syncwarp after its last slab store: the vector is visible)
                        bat_rescale(bp.phit[k] + inst * bp.N, bp.N, bp.P, resc, lane);
                        __syncwarp();
#pragma unroll
                        for (int q = 0; q < L; ++q)
                            if (q == k) {
                                E[q] = -sumE + shk + resc;
                                Sh[q] = shk + resc;
                            }
                    } else if (!upd) {
                        res += acc;
                    }
                }
                __syncthreads();
                // chain operators of the next slot's bound set
                const int nk = sl + 1 < nslots ? ((sl + 1) < L ? sl + 1 : sl + 1 - L + roff) : 0;
                if (live) bat_ops<NB, T, PTS>(bp, inst, nk, wt, buf, ops, lane);
                __syncthreads();
            }
            if (live) {
                done_it = t;
                if (check) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) res += __shfl_xor_sync(0xffffffffu, res, o);
                    if (defer) {
                        pend = true;
                        pres = res;
                        pt = t;
                    } else {
                        last_res = res;
                        if (res <= bp.tol) conv = true;
                    }
                }
            }
        }
        if (active) {
#pragma unroll
            for (int q = 0; q < L; ++q) bp.E[(inst * L + q) * 32 + lane] = E[q];
            const bool anybad = __any_sync(0xffffffffu, bad);
            int fi = fail;
            for (int o = 16; o > 0; o >>= 1) fi = max(fi, __shfl_down_sync(0xffffffffu, fi, o));
            if (lane == 0) {
                bp.status[inst] = anybad ? 6 : 0;
                bp.fail_iter[inst] = anybad ? fi : -1;
                bp.iters_done[inst] = done_it;
                bp.converged[inst] = conv ? 1 : 0;
                bp.resid[inst] = last_res;
            }
        }
    }
}

// One product of mode MARG (out = m_k) or COST (wout = W) for every instance.
template <int NB, typename T, int MODE, bool PTS>
__global__ void __launch_bounds__(kBWarps * 32) k_bat_product(BPlan bp) {
    constexpr int L = NB + 1;
    constexpr int M = 1 << NB;
    constexpr int S = kBS;
    constexpr int TILE = 32 * (S + 1);
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t slot = (int64_t)blockIdx.x * kBWarps + warp;
    double *buf = smem + (size_t)warp * (2 * L + 1) * TILE;
    T *ops = reinterpret_cast<T *>(bp.ops) + slot * 2 * OpShape<NB>::SZ * 32;
    T *ck = reinterpret_cast<T *>(bp.ckpt) + slot * (int64_t)(bp.P / S) * M * 32;
    const int k = bp.k;
    for (int64_t inst = slot; inst < bp.batch; inst += bp.slots) {
        double w0[NB + 2];
        bweights<NB>(w0, bp.eta[inst], bp.h);
        T wt[NB + 2];
#pragma unroll
        for (int a = 0; a <= NB + 1; ++a) {
            if constexpr (sizeof(T) == sizeof(double)) {
                reinterpret_cast<double &>(wt[a]) = w0[a];
            } else {
                const double e = a <= L ? (double)(a * (L - a)) : 0.0;
                reinterpret_cast<Dual &>(wt[a]) = Dual{w0[a], e * w0[a]};
            }
        }
        int E[kMaxL];
#pragma unroll
        for (int q = 0; q < kMaxL; ++q) E[q] = q < L ? bp.E[(inst * L + q) * 32 + lane] : 0;
        bat_ops<NB, T, PTS>(bp, inst, k, wt, buf, ops, lane);
        T F[M], B[M];
        if (31 * (int64_t)bp.P < bp.N) bat_carries<NB, T, true>(ops, k, E, F, B, lane, bp);
        else bat_carries<NB, T, false>(ops, k, E, F, B, lane, bp);
        bat_walk1<NB, T, PTS>(bp, inst, k, wt, B, buf, ck, lane);
        int sumE = 0;
#pragma unroll
        for (int q = 0; q < L; ++q)
            if (q != k) sumE += E[q];
        int Ek = 0;
#pragma unroll
        for (int q = 0; q < L; ++q)
            if (q == k) Ek = E[q];
        double acc = 0.0;
        bool bad = false;
        bat_walk2<NB, T, MODE, (sizeof(T) == sizeof(double) ? 4 : 2), PTS>(bp, inst, k, wt, F, buf, ck, sumE, Ek, acc, bad, lane);
        if (MODE == MODE_COST) {
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
            if (lane == 0) bp.wout[inst] = bp.hc * acc;
        }
    }
}

// Segmented fill across the warp: lanes without mass take e of the nearest lane with mass to
// the left, or (none to the left) to the right.
__device__ __forceinline__ int fill_exponent(int e, bool has, int lane) {
    const int NONE = -2147483647;
    int v = has ? e : NONE;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d && v == NONE) v = o;
    }
    int w = has ? e : NONE;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_down_sync(0xffffffffu, w, d);
        if (lane + d < 32 && w == NONE) w = o;
    }
    return v != NONE ? v : (w != NONE ? w : 0);
}

// log phi (natural [batch][N] planes) -> mantissas + chain exponents; one warp per instance.
__global__ void k_bat_import(BPlan bp, const double *const *u, int is_log) {
    const int lane = threadIdx.x & 31;
    const int64_t inst = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (inst >= bp.batch) return;
    const int64_t x0 = (int64_t)lane * bp.P, x1 = min(bp.N, x0 + bp.P);
    for (int q = 0; q < bp.l; ++q) {
        const double *g = u[q] + inst * bp.N;
        double *o = bp.phit[q] + inst * bp.N;
        int e;
        bool has_mass;
        if (is_log) {
            double gm = -INFINITY;
            for (int64_t x = x0; x < x1; ++x) gm = fmax(gm, g[x]);
            has_mass = isfinite(gm);
            e = has_mass ? (int)floor(gm * 1.4426950408889634) : 0;
            const double off = (double)e * 0.6931471805599453;
            for (int64_t x = x0; x < x1; ++x) o[x] = exp(g[x] - off);
        } else {
            int em = -1000000;
            for (int64_t x = x0; x < x1; ++x)
                if (g[x] > 0) em = max(em, ilog2d(g[x]));
            has_mass = em > -1000000;
            e = has_mass ? em : 0;
            const double sc = pow2i(-e);
            for (int64_t x = x0; x < x1; ++x) o[x] = g[x] * sc;
        }
        // chains without mass (all phi = 0, or beyond N) take the exponent of the nearest chain
        // with mass to the left (else to the right): the carries then cross them unscaled
        bp.E[(inst * bp.l + q) * 32 + lane] = fill_exponent(e, has_mass, lane);
    }
}

__global__ void k_bat_export(BPlan bp, double *const *u, int is_log) {
    const int lane = threadIdx.x & 31;
    const int64_t inst = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (inst >= bp.batch) return;
    const int64_t x0 = (int64_t)lane * bp.P, x1 = min(bp.N, x0 + bp.P);
    for (int q = 0; q < bp.l; ++q) {
        const double *m = bp.phit[q] + inst * bp.N;
        double *o = u[q] + inst * bp.N;
        const int e = bp.E[(inst * bp.l + q) * 32 + lane];
        if (is_log) {
            const double off = (double)e * 0.6931471805599453;
            for (int64_t x = x0; x < x1; ++x) o[x] = log(m[x]) + off;
        } else {
            for (int64_t x = x0; x < x1; ++x) o[x] = scale2(m[x], e);
        }
    }
}

// Smallest per-instance mass of one marginal plane [batch][N] (EZEROMASS per instance):
// one warp per instance, atomicMin on the bit pattern (order-preserving for non-negative
// doubles; negative sums are reported as ENEGMASS by the element check first).
__global__ void k_bat_min_mass(const double *mu, int64_t batch, int64_t N, double *mass) {
    const int lane = threadIdx.x & 31;
    const int64_t inst = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (inst >= batch) return;
    double sum = 0.0;
    for (int64_t x = lane; x < N; x += 32) sum += mu[inst * N + x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) atomicMin(reinterpret_cast<unsigned long long *>(mass), (unsigned long long)__double_as_longlong(fmax(sum, 0.0)));
}

cudaError_t launch_bat_min_mass(const double *mu, int64_t batch, int64_t N, double *mass, cudaStream_t s,
                                int64_t *launches) {
    cudaMemsetAsync(mass, 0x7f, sizeof(double), s);  // 1.4e306: larger than any mass
    k_bat_min_mass<<<(unsigned)((batch + 3) / 4), 128, 0, s>>>(mu, batch, N, mass);
    ++*launches;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
template <int NB>
static size_t bat_smem() {
    return (size_t)kBWarps * (2 * (NB + 1) + 1) * 32 * (kBS + 1) * sizeof(double);
}

int64_t bat_slots(int l) {
    if (const char *e = getenv("MMOT_BAT_SLOTS")) return atoll(e);  // experiments only
    int n = 0;
    const int NB = l - 1;
    auto q = [&](auto kern, size_t sm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kBWarps * 32, sm);
    };
    switch (NB) {
        case 1: q(k_bat_sinkhorn<1, false, false>, bat_smem<1>()); break;
        case 2: q(k_bat_sinkhorn<2, false, false>, bat_smem<2>()); break;
        case 3: q(k_bat_sinkhorn<3, false, false>, bat_smem<3>()); break;
        case 4: q(k_bat_sinkhorn<4, false, false>, bat_smem<4>()); break;
        default: n = 1;
    }
    cudaGetLastError();
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (int64_t)nsm * (n > 0 ? n : 1) * kBWarps;
}

static BPlan to_bplan(const BatchArgs &a) {
    BPlan bp{};
    bp.l = a.l;
    bp.N = a.N;
    bp.batch = a.batch;
    bp.P = a.P;
    bp.h = a.h;
    bp.eta = a.eta;
    for (int q = 0; q < kMaxL; ++q) {
        bp.phit[q] = a.phit[q];
        bp.mu[q] = a.mu[q];
    }
    bp.E = a.E;
    bp.ops = a.ops;
    bp.ckpt = a.ckpt;
    bp.rsave = a.rsave;
    bp.lam = a.lam;
    bp.hx = a.hx;
    bp.ne = a.ne;
    bp.hc = a.lam ? 1.0 : a.h;
    bp.slots = a.slots;
    bp.iters = a.iters;
    bp.k = a.k;
    bp.out = a.out;
    bp.wout = a.wout;
    bp.status = a.status;
    bp.fail_iter = a.fail_iter;
    bp.renorm = g_renorm;
    bp.tol = a.tol;
    bp.check_every = a.check_every > 0 ? a.check_every : 1;
    bp.iters_done = a.iters_done;
    bp.converged = a.converged;
    bp.resid = a.resid;
    return bp;
}

template <int NB, bool PTS>
static cudaError_t bat_run(const BatchArgs &a, int what, cudaStream_t s, int64_t *launches) {
    const BPlan bp = to_bplan(a);
    const unsigned grid = (unsigned)((a.slots + kBWarps - 1) / kBWarps);
    const size_t sm = bat_smem<NB>();
    switch (what) {
        case 0:
            smem_attr((const void *)k_bat_sinkhorn<NB, PTS, false>, sm);
            smem_attr((const void *)k_bat_sinkhorn<NB, PTS, true>, sm);
            if (a.tol > 0) k_bat_sinkhorn<NB, PTS, true><<<grid, kBWarps * 32, sm, s>>>(bp);
            else k_bat_sinkhorn<NB, PTS, false><<<grid, kBWarps * 32, sm, s>>>(bp);
            break;
        case 1:
            smem_attr((const void *)k_bat_product<NB, double, MODE_MARG, PTS>, sm);
            k_bat_product<NB, double, MODE_MARG, PTS><<<grid, kBWarps * 32, sm, s>>>(bp);
            break;
        default:
            smem_attr((const void *)k_bat_product<NB, Dual, MODE_COST, PTS>, sm);
            k_bat_product<NB, Dual, MODE_COST, PTS><<<grid, kBWarps * 32, sm, s>>>(bp);
            break;
    }
    ++*launches;
    return cudaGetLastError();
}

template <int NB>
static cudaError_t bat_run_any(const BatchArgs &a, int what, cudaStream_t s, int64_t *launches) {
    return a.lam ? bat_run<NB, true>(a, what, s, launches) : bat_run<NB, false>(a, what, s, launches);
}

cudaError_t launch_batched(const BatchArgs &a, int what, cudaStream_t s, int64_t *launches) {
    switch (a.l - 1) {
        case 1: return bat_run_any<1>(a, what, s, launches);
        case 2: return bat_run_any<2>(a, what, s, launches);
        case 3: return bat_run_any<3>(a, what, s, launches);
        case 4: return bat_run_any<4>(a, what, s, launches);
        default: return cudaErrorInvalidValue;
    }
}

// lambda_e = exp(-h_e / eta_b) for every instance b and edge e (1 for edges outside the grid).
__global__ void k_bat_lambda(double *lam, const double *hx, const double *eta, int64_t batch, int64_t ne) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch * ne) return;
    const int64_t b = i / ne, e = i % ne;
    const double h = hx[e];
    lam[i] = h > 0.0 ? exp(-h / eta[b]) : 1.0;
}

cudaError_t launch_bat_lambda(double *lam, const double *hx, const double *eta, int64_t batch, int64_t ne, cudaStream_t s) {
    const int64_t n = batch * ne;
    k_bat_lambda<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lam, hx, eta, batch, ne);
    return cudaGetLastError();
}

cudaError_t launch_bat_convert(const BatchArgs &a, void *const *u_dev_ptrs, int import, int is_log, cudaStream_t s,
                               int64_t *launches) {
    const BPlan bp = to_bplan(a);
    const unsigned grid = (unsigned)((a.batch + 3) / 4);
    if (import) k_bat_import<<<grid, 128, 0, s>>>(bp, reinterpret_cast<const double *const *>(u_dev_ptrs), is_log);
    else k_bat_export<<<grid, 128, 0, s>>>(bp, reinterpret_cast<double *const *>(u_dev_ptrs), is_log);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace mmot
