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
// Layout / parallelism: one warp per instance, lane S = subset state S (2^(l-1) <= 32 lanes), the
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
template <bool TAN>
__device__ double st_product(const SPlan &sp, int64_t b, int k, int mode, bool &bad, int lane) {
    const int l = sp.l, NB = l - 1, M = 1 << NB;
    const int64_t N = sp.N;
    const double eta = sp.eta[b];
    double lw[kMaxL + 2], le[kMaxL + 2];
#pragma unroll
    for (int a = 0; a <= kMaxL + 1; ++a) {
        const double e = a <= l ? (double)(a * (l - a)) : 0.0;
        lw[a] = a <= l ? -e * sp.h / eta : -INFINITY;
        le[a] = e > 0 ? log(e) : -INFINITY;
    }
    const double *gq[kMaxL];
    for (int j = 0; j < NB; ++j) gq[j] = sp.g[(k + 1 + j) % l] + b * N;
    double *gk = sp.g[k] + b * N;
    const double *muk = sp.mu[k] ? sp.mu[k] + b * N : nullptr;
    // this warp's slot of prefix-state storage ([2][N][M]: states, tangents)
    double *pre = sp.scratch + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * sp.scratch_per_warp;
    const bool act = lane < M;
    const int S = lane & (M - 1);
    const int pcS = __popc(S);
    // prefix walk: store F (and hatF) of every point
    double F = S == 0 ? 0.0 : -INFINITY, Fh = -INFINITY;
    for (int64_t x = 0; x < N; ++x) {
        const double a = lw[pcS];
        if (TAN) Fh = lae(Fh + a, F + a + le[pcS]);
        F += a;
        for (int j = 0; j < NB; ++j) {
            const double gx = gq[j][x];  // plain load: g is rewritten inside the launch
            const double o = __shfl_xor_sync(0xffffffffu, F, 1 << j);
            const double oh = TAN ? __shfl_xor_sync(0xffffffffu, Fh, 1 << j) : 0.0;
            if ((S >> j) & 1) {
                F = lae(F, gx + o);
                if (TAN) Fh = lae(Fh, gx + oh);
            }
        }
        if (act) {
            pre[x * M + S] = F;
            if (TAN) pre[(N + x) * M + S] = Fh;
        }
    }
    __syncwarp();
    // suffix walk with the combine at every point
    double B = S == 0 ? 0.0 : -INFINITY, Bh = -INFINITY;
    double acc = 0.0;
    const int full = M - 1;
    for (int64_t x = N - 1; x >= 0; --x) {
        // B holds B_{x+1}; combine J_x = sum_S F_x[S] w_{|S|+1} B_{x+1}[S^c]
        const double Bc = __shfl_sync(0xffffffffu, B, full & ~S);
        const double Fx = act ? pre[x * M + S] : -INFINITY;
        double term = act ? Fx + lw[pcS + 1] + Bc : -INFINITY;
        if (TAN) {
            const double Bhc = __shfl_sync(0xffffffffu, Bh, full & ~S);
            const double Fhx = act ? pre[(N + x) * M + S] : -INFINITY;
            term = act ? lae(lae(Fhx + lw[pcS + 1] + Bc, Fx + lw[pcS + 1] + le[pcS + 1] + Bc), Fx + lw[pcS + 1] + Bhc)
                       : -INFINITY;
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
        const double a = lw[pcS];
        if (TAN) Bh = lae(Bh + a, B + a + le[pcS]);
        B += a;
        for (int j = 0; j < NB; ++j) {
            const double gx = gq[j][x];  // plain load: g is rewritten inside the launch
            const double o = __shfl_xor_sync(0xffffffffu, B, 1 << j);
            const double oh = TAN ? __shfl_xor_sync(0xffffffffu, Bh, 1 << j) : 0.0;
            if ((S >> j) & 1) {
                B = lae(B, gx + o);
                if (TAN) Bh = lae(Bh, gx + oh);
            }
        }
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, acc, 0);
}

// what: 0 Sinkhorn, 1 marginal k -> out, 2 cost -> wout.  One warp per instance (grid-stride).
__global__ void __launch_bounds__(128) k_stable(SPlan sp, int what) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = w0; b < sp.batch; b += nw) {
        if (sp.status[b] || (sp.sel && !sp.sel[b])) continue;
        bool bad = false;
        if (what == 1) {
            st_product<false>(sp, b, sp.k, MODE_MARG, bad, lane);
            continue;
        }
        if (what == 2) {
            const double acc = st_product<true>(sp, b, sp.l - 1, MODE_COST, bad, lane);
            if (lane == 0) sp.wout[b] = sp.hc * acc;
            continue;
        }
        int t = 0;
        double res = NAN;
        bool conv = false;
        while (t < sp.iters) {
            ++t;
            for (int k = 0; k < sp.l && !bad; ++k) st_product<false>(sp, b, k, MODE_UPD, bad, lane);
            bad = __any_sync(0xffffffffu, bad);
            if (bad) break;
            if (sp.tol > 0 && (t % sp.check_every == 0 || t == sp.iters)) {
                double r = 0.0;
                for (int k = 0; k + 1 < sp.l; ++k) r += st_product<false>(sp, b, k, MODE_RES, bad, lane);
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
    k_stable<<<blocks, 128, 0, s>>>(sp, what);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace mmot
