// stable.cu -- the stabilised kernel family (MMOT_KERNEL_STABLE): the subset-lattice recurrence of
// dp.cuh evaluated in the LOG domain, for scalings and products beyond fp64's range (a8).
//
// The paper's remedy for over/underflow is log-domain stabilisation: absorb the potentials into the
// kernel (Remark 1) and run the recursions on the absorbed quantities (Algorithm 5,
// FTVP-LOG), without which its own solver dies at iteration 89.  Here every
// prefix / suffix state is carried as its logarithm, so a state may be e^-8000 next to a state of
// e^+4000 (disjoint supports at eta = 1e-4: crossing a gap of 0.4 costs e^-0.8/eta):
//     diag:    F[S] += log w_{|S|}                       (w_a = lambda^{a(l-a)})
//     place:   F[S] = logaddexp(F[S], g_q[x] + F[S \ q]) (in place, q over the bound marginals)
//     combine: log J_k[m] = logsumexp_S (F_m[S] + log w_{|S|+1} + B_{m+1}[S^c])
// and the Sinkhorn update is g_k = log mu_k - log J_k with g = log phi.  The cost
// tangent hatJ = sum E lambda^E prod phi is carried as the log of the E-weighted sums
// (d/dlog lambda of w_a is e_a w_a).
//
// Layout / parallelism: one warp per instance, lane S = subset state S (2^(l-1) <= 32 lanes; for
// l = 7, 8 each lane holds 2 / 4 states, S = lane | r << 5), the
// grid walked sequentially (prefix walk storing every prefix state, then the suffix walk with the
// combine).  O(N) work like the plain families but O(N) latency per product and ~50 fp64
// instructions per logaddexp: this is the robust family the plain ones fall back to when a product
// leaves the fp64 range (MMOT_EOVERFLOW), not the fast path.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "internal.h"

namespace mmot {

__device__ __forceinline__ double lae(double a, double b) {  // log(e^a + e^b), -inf safe
    const double m = fmax(a, b);
    if (m == -INFINITY) return -INFINITY;
    return m + log1p(exp(-fabs(a - b)));
}

// warp-wide logsumexp over lanes 0..M-1 (M a power of two; other lanes hold -inf)
__device__ __forceinline__ double warp_lse(double v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = lae(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// One product J_k (or hatJ_k) of instance b; returns per-mode reductions.
//   UPD : g_k[x] = log mu_k[x] - log J_k[x]                (bad: J not finite where mu > 0)
//   MARG: out[x] = exp(g_k[x] + log J_k[x])
//   RES : returns sum_x |exp(g_k + log J_k) - mu_k|
//   COST: returns sum_x exp(g_k + log hatJ_k)  (times hc by the caller)
// R states per lane: state S = lane | r << 5 (R = 1 for l <= 6; R = 2, 4 for l = 7, 8, where the
// bound marginals j >= 5 pair registers of the same lane instead of lanes).
template <int R, bool TAN>
__device__ double st_product(const SPlan &sp, int64_t b, int k, int mode, bool &bad, int lane) {
    const int l = sp.l, NB = l - 1, M = 1 << NB;
    const int NBL = NB < 5 ? NB : 5;  // bound marginals on lane bits
    const int64_t N = sp.N;
    const double eta = sp.eta[b];
    double lw[kStMaxL + 2], le[kStMaxL + 2];
#pragma unroll
    for (int a = 0; a <= kStMaxL + 1; ++a) {
        const double e = a <= l ? (double)(a * (l - a)) : 0.0;
        lw[a] = a <= l ? -e * sp.h / eta : -INFINITY;
        le[a] = e > 0 ? log(e) : -INFINITY;
    }
    const double *gq[kStMaxL];
    for (int j = 0; j < NB; ++j) gq[j] = sp.g[(k + 1 + j) % l] + b * N;
    double *gk = sp.g[k] + b * N;
    const double *muk = sp.mu[k] ? sp.mu[k] + b * N : nullptr;
    // this warp's slot of prefix-state storage ([2][N][M]: states, tangents)
    double *pre = sp.scratch + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * sp.scratch_per_warp;
    const bool act = R > 1 || lane < M;
    const int SL = R > 1 ? lane : lane & (M - 1);  // lane part of the state index
    const int pcL = __popc(SL);
    // prefix walk: store F (and hatF) of every point
    double F[R], Fh[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        F[r] = (SL == 0 && r == 0) ? 0.0 : -INFINITY;
        Fh[r] = -INFINITY;
    }
    for (int64_t x = 0; x < N; ++x) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pc = pcL + __popc(r);
            const double a = lw[pc];
            if (TAN) Fh[r] = lae(Fh[r] + a, F[r] + a + le[pc]);
            F[r] += a;
        }
        for (int j = 0; j < NBL; ++j) {
            const double gx = gq[j][x];  // plain load: g is rewritten inside the launch
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double o = __shfl_xor_sync(0xffffffffu, F[r], 1 << j);
                const double oh = TAN ? __shfl_xor_sync(0xffffffffu, Fh[r], 1 << j) : 0.0;
                if ((SL >> j) & 1) {
                    F[r] = lae(F[r], gx + o);
                    if (TAN) Fh[r] = lae(Fh[r], gx + oh);
                }
            }
        }
        if (R > 1) {
#pragma unroll
            for (int jb = 0; jb < 2; ++jb) {
                if ((1 << jb) < R) {
                    const double gx = gq[5 + jb][x];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if ((r >> jb) & 1) {
                            F[r] = lae(F[r], gx + F[r ^ (1 << jb)]);
                            if (TAN) Fh[r] = lae(Fh[r], gx + Fh[r ^ (1 << jb)]);
                        }
                }
            }
        }
        if (act) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                pre[x * M + SL + 32 * r] = F[r];
                if (TAN) pre[(N + x) * M + SL + 32 * r] = Fh[r];
            }
        }
    }
    __syncwarp();
    // suffix walk with the combine at every point
    double B[R], Bh[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        B[r] = (SL == 0 && r == 0) ? 0.0 : -INFINITY;
        Bh[r] = -INFINITY;
    }
    double acc = 0.0;
    const int cl = (R > 1 ? 31 : M - 1) & ~SL;  // lane holding the complement's lane part
    for (int64_t x = N - 1; x >= 0; --x) {
        // B holds B_{x+1}; combine J_x = sum_S F_x[S] w_{|S|+1} B_{x+1}[S^c]
        double term = -INFINITY;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pc = pcL + __popc(r);
            const double Bc = __shfl_sync(0xffffffffu, B[R - 1 - r], cl);
            const double Fx = act ? pre[x * M + SL + 32 * r] : -INFINITY;
            double t = act ? Fx + lw[pc + 1] + Bc : -INFINITY;
            if (TAN) {
                const double Bhc = __shfl_sync(0xffffffffu, Bh[R - 1 - r], cl);
                const double Fhx = act ? pre[(N + x) * M + SL + 32 * r] : -INFINITY;
                t = act ? lae(lae(Fhx + lw[pc + 1] + Bc, Fx + lw[pc + 1] + le[pc + 1] + Bc), Fx + lw[pc + 1] + Bhc)
                        : -INFINITY;
            }
            term = R > 1 ? lae(term, t) : t;
        }
        const double lj = warp_lse(term);
        if (lane == 0) {
            if (mode == MODE_UPD) {
                const double m = __ldg(muk + x);
                const double gnew = m > 0.0 ? log(m) - lj : -INFINITY;
                bad |= m > 0.0 && !isfinite(gnew);
                gk[x] = gnew;
            } else if (mode == MODE_MARG) {
                sp.out[b * N + x] = exp(gk[x] + lj);
            } else if (mode == MODE_RES) {
                acc += fabs(exp(gk[x] + lj) - __ldg(muk + x));
            } else {
                acc += exp(gk[x] + lj);
            }
        }
        // B_x = place_x(diag B_{x+1})
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pc = pcL + __popc(r);
            const double a = lw[pc];
            if (TAN) Bh[r] = lae(Bh[r] + a, B[r] + a + le[pc]);
            B[r] += a;
        }
        for (int j = 0; j < NBL; ++j) {
            const double gx = gq[j][x];  // plain load: g is rewritten inside the launch
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double o = __shfl_xor_sync(0xffffffffu, B[r], 1 << j);
                const double oh = TAN ? __shfl_xor_sync(0xffffffffu, Bh[r], 1 << j) : 0.0;
                if ((SL >> j) & 1) {
                    B[r] = lae(B[r], gx + o);
                    if (TAN) Bh[r] = lae(Bh[r], gx + oh);
                }
            }
        }
        if (R > 1) {
#pragma unroll
            for (int jb = 0; jb < 2; ++jb) {
                if ((1 << jb) < R) {
                    const double gx = gq[5 + jb][x];
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if ((r >> jb) & 1) {
                            B[r] = lae(B[r], gx + B[r ^ (1 << jb)]);
                            if (TAN) Bh[r] = lae(Bh[r], gx + Bh[r ^ (1 << jb)]);
                        }
                }
            }
        }
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, acc, 0);
}

// what: 0 Sinkhorn, 1 marginal k -> out, 2 cost -> wout.  One warp per instance (grid-stride).
template <int R>
__global__ void __launch_bounds__(128) k_stable(SPlan sp, int what) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = w0; b < sp.batch; b += nw) {
        if (sp.status[b] || (sp.sel && !sp.sel[b])) continue;
        bool bad = false;
        if (what == 1) {
            st_product<R, false>(sp, b, sp.k, MODE_MARG, bad, lane);
            continue;
        }
        if (what == 2) {
            const double acc = st_product<R, true>(sp, b, sp.l - 1, MODE_COST, bad, lane);
            if (lane == 0) sp.wout[b] = sp.hc * acc;
            continue;
        }
        int t = 0;
        double res = NAN;
        bool conv = false;
        while (t < sp.iters) {
            ++t;
            for (int k = 0; k < sp.l && !bad; ++k) st_product<R, false>(sp, b, k, MODE_UPD, bad, lane);
            bad = __any_sync(0xffffffffu, bad);
            if (bad) break;
            if (sp.tol > 0 && (t % sp.check_every == 0 || t == sp.iters)) {
                double r = 0.0;
                for (int k = 0; k + 1 < sp.l; ++k) r += st_product<R, false>(sp, b, k, MODE_RES, bad, lane);
                res = r;
                if (r <= sp.tol) {
                    conv = true;
                    break;
                }
            }
        }
        if (lane == 0) {
            if (bad) {
                sp.status[b] = 6;  // EOVERFLOW (a product left even the log domain: NaN / zero kernel)
                sp.fail_iter[b] = t;
            }
            sp.iters_done[b] = bad ? t - 1 : t;
            sp.converged[b] = conv ? 1 : 0;
            sp.resid[b] = res;
        }
    }
}

// u (caller layout, LOG or LINEAR) <-> g = log phi, for the instances selected by sel (all if null)
__global__ void k_st_convert(const double *__restrict__ in, double *__restrict__ out, int64_t batch, int64_t N,
                             const int *sel, int to_log) {
    const int64_t n = batch * N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (sel && !sel[i / N]) continue;
        const double v = in[i];
        out[i] = to_log ? log(v) : exp(v);
    }
}
__global__ void k_st_copy(const double *__restrict__ in, double *__restrict__ out, int64_t batch, int64_t N,
                          const int *sel) {
    const int64_t n = batch * N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!sel || sel[i / N]) out[i] = in[i];
}

cudaError_t launch_st_convert(const double *in, double *out, int64_t batch, int64_t N, const int *sel, int op,
                              cudaStream_t s, int64_t *launches) {
    const int64_t n = batch * N;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    if (op == 0) k_st_copy<<<grid, 256, 0, s>>>(in, out, batch, N, sel);
    else k_st_convert<<<grid, 256, 0, s>>>(in, out, batch, N, sel, op == 1 ? 1 : 0);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_stable(const SPlan &sp, int what, cudaStream_t s, int64_t *launches) {
    const int64_t warps = std::min<int64_t>(sp.batch, sp.slots);
    const unsigned blocks = (unsigned)((warps + 3) / 4);
    if (sp.l <= 6) k_stable<1><<<blocks, 128, 0, s>>>(sp, what);
    else if (sp.l == 7) k_stable<2><<<blocks, 128, 0, s>>>(sp, what);
    else k_stable<4><<<blocks, 128, 0, s>>>(sp, what);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace mmot
