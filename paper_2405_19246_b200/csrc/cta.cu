// cta.cu -- the CTA family: one thread block per small instance (BASELINE C1: l = 3, N = 64;
// C2: l = 4, N = 1000, tol = 1e-9), every sweep of the solve inside one launch.
//
// The persistent batched kernel (batched.cu) gives an instance one warp: 32 chains, each walked
// serially, the chain operators joined by a 31-step serial carry propagation per direction -- a
// single warp of a single SM does all of C2's 6 000 products (ncu: 98 % of the samples are the other
// seven warps waiting at the CTA barrier).  Here the instance gets a whole CTA of 256 threads:
//   chains   thread c owns points [cP, (c+1)P), P = ceil(N / 256) rounded up to a power of two
//            (the grid is zero-padded to 256 P points: a zero scaling places nothing, and the
//            padding sits beyond the last point, where only states nobody reads depend on it)
//   ops      each thread walks its chain once (extended walk, dp.cuh opx_*): prefix and suffix
//            operators of the update's bound set
//   scan     Kogge-Stone over the 32 lanes of each warp by operator composition (dp.cuh op_compose,
//            5 levels per direction), the 8 warp aggregates through shared memory, the carries
//            entering each chain = the exclusive composite applied to the state entering its warp
//   walks    suffix walk with sub-block checkpoints (registers), prefix walk with the sub-block
//            suffix states rebuilt, combine J_k = sum_S F[S] w_{|S|+1} B[S^c], phi_k = mu_k / J_k
// with two CTA barriers per product.  Scalings are plain fp64 (no exponents): the family is used
// when (l-1) * (x_max - x_min) / eta <= kCtaRange for every instance, i.e. |log phi| stays far
// inside fp64's range; products that still leave it report EOVERFLOW and the batched driver redoes
// the instance on the stabilised family (api.cu bat_sinkhorn).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "internal.h"
#include "walk.cuh"

namespace mmot {

constexpr int kCtaT = 256;  // threads (chains) per instance
constexpr int kCtaW = kCtaT / 32;

template <int NB>
struct CtaOp {
    static constexpr int M = 1 << NB;
};

// shuffle every used entry of an operator (entries with |V| > NB - c are identically zero)
template <int NB>
__device__ __forceinline__ void op_shfl_up(double (&D)[NB + 1][1 << NB], const double (&G)[NB + 1][1 << NB], int d) {
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int V = 0; V < (1 << NB); ++V)
            D[c][V] = pc(V) <= NB - c ? __shfl_up_sync(0xffffffffu, G[c][V], d) : 0.0;
}
template <int NB>
__device__ __forceinline__ void op_shfl_down(double (&D)[NB + 1][1 << NB], const double (&G)[NB + 1][1 << NB], int d) {
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int V = 0; V < (1 << NB); ++V)
            D[c][V] = pc(V) <= NB - c ? __shfl_down_sync(0xffffffffu, G[c][V], d) : 0.0;
}

// One product of update / residual slot k for the block's instance.
//   MODE_UPD: phi_k <- mu_k / J_k;  MODE_RES: returns this thread's sum |phi_k J_k - mu_k|
//   DEFER (MODE_UPD, k = 0 after a check sweep): the new phi_0 goes to cp.scr and the product also
//   returns the deferred residual term |phi_0 J_0 - mu_0| of the previous sweep (same bound vectors)
template <int NB, int P, int MODE, bool DEFER = false>
__device__ __forceinline__ double cta_product(const CtaPlan &cp, int64_t inst, int k, const double (&wt)[NB + 2],
                                              double (*aggF)[(NB + 1) << NB], double (*aggB)[(NB + 1) << NB],
                                              bool &bad) {
    constexpr int L = NB + 1, M = 1 << NB, SZ = (NB + 1) * M;
    constexpr int Q = P < 4 ? P : 4, NQ = P / Q;
    const int c = threadIdx.x, lane = c & 31, w = c >> 5;
    const int64_t N = cp.N;
    const int64_t x0 = (int64_t)c * P;
    const double *vb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) vb[b] = cp.phi[(k + 1 + b) % L] + inst * N;
    auto fval = [&](double (&f)[NB > 0 ? NB : 1], int j) {
        const int64_t x = x0 + j;
#pragma unroll
        for (int b = 0; b < NB; ++b) f[b] = x < N ? vb[b][x] : 0.0;
    };
    // ---- chain operators (extended walk)
    double pf[SZ], pb[SZ];
    {
        double G[NB + 1][M];
        opx_identity<NB, double>(G);
#pragma unroll
        for (int j = 0; j < P; ++j) {
            double f[NB > 0 ? NB : 1];
            fval(f, j);
            opx_step<NB, double>(G, wt, f, j == 0);
        }
#pragma unroll
        for (int i = 0; i < SZ; ++i) pf[i] = pb[i] = 0.0;
        opx_store<NB, double>(G, wt, pf, pb);
    }
    // ---- prefix direction: inclusive warp scan, warp aggregate, exclusive composite of the lane
    double Ex[NB + 1][M];
    {
        double Gp[NB + 1][M], D[NB + 1][M], C[NB + 1][M];
        op_load<NB, double>(Gp, pf);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            op_shfl_up<NB>(D, Gp, d);
            op_compose<NB, double>(D, Gp, C);  // earlier chains first
            if (lane >= d) {
#pragma unroll
                for (int cc = 0; cc <= NB; ++cc)
#pragma unroll
                    for (int V = 0; V < M; ++V) Gp[cc][V] = C[cc][V];
            }
        }
        if (lane == 31) op_store<NB, double>(Gp, aggF[w]);
        op_shfl_up<NB>(Ex, Gp, 1);
        if (lane == 0) op_identity<NB, double>(Ex);
    }
    double Exs[NB + 1][M];
    {
        double Gs[NB + 1][M], D[NB + 1][M], C[NB + 1][M];
        op_load<NB, double>(Gs, pb);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            op_shfl_down<NB>(D, Gs, d);
            op_compose<NB, double>(D, Gs, C);  // later chains first
            if (lane + d < 32) {
#pragma unroll
                for (int cc = 0; cc <= NB; ++cc)
#pragma unroll
                    for (int V = 0; V < M; ++V) Gs[cc][V] = C[cc][V];
            }
        }
        if (lane == 0) op_store<NB, double>(Gs, aggB[w]);
        op_shfl_down<NB>(Exs, Gs, 1);
        if (lane == 31) op_identity<NB, double>(Exs);
    }
    __syncthreads();
    // ---- carries: the states entering this warp (from the warp aggregates), then this chain's
    double Fin[M], Bend[M];
    {
        double v[M], y[M], G[NB + 1][M];
        vec_unit<NB, double>(v);
        for (int ww = 0; ww < w; ++ww) {
            op_load<NB, double>(G, aggF[ww]);
            op_apply<NB, double>(G, v, y);
#pragma unroll
            for (int S = 0; S < M; ++S) v[S] = y[S];
        }
        op_apply<NB, double>(Ex, v, Fin);
        vec_unit<NB, double>(v);
        for (int ww = kCtaW - 1; ww > w; --ww) {
            op_load<NB, double>(G, aggB[ww]);
            op_apply<NB, double>(G, v, y);
#pragma unroll
            for (int S = 0; S < M; ++S) v[S] = y[S];
        }
        op_apply<NB, double>(Exs, v, Bend);
    }
    // ---- walk 1 (right to left): suffix state after every sub-block
    double ck[NQ][M];
    {
        double st[M];
#pragma unroll
        for (int S = 0; S < M; ++S) st[S] = Bend[S];
#pragma unroll
        for (int q = NQ - 1; q >= 0; --q) {
#pragma unroll
            for (int S = 0; S < M; ++S) ck[q][S] = st[S];
            if (q > 0) {
#pragma unroll
                for (int i = Q - 1; i >= 0; --i) {
                    double f[NB > 0 ? NB : 1];
                    fval(f, q * Q + i);
                    dp_diag<NB, double, true>(st, wt);
                    dp_place<NB, double>(st, f);
                }
            }
        }
    }
    // ---- walk 2 (left to right): prefix states, sub-block suffix states rebuilt, combine
    double acc = 0.0;
    double *phik = cp.phi[k] + inst * N;
    const double *muk = cp.mu[k] + inst * N;
    double F[M];
#pragma unroll
    for (int S = 0; S < M; ++S) F[S] = Fin[S];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double H[Q][M], st[M];
#pragma unroll
        for (int S = 0; S < M; ++S) st[S] = ck[q][S];
#pragma unroll
        for (int i = Q - 1; i >= 0; --i) {
            dp_diag<NB, double, true>(st, wt);  // H_x = D B_{x+1}
#pragma unroll
            for (int S = 0; S < M; ++S) H[i][S] = st[S];
            if (i > 0) {
                double f[NB > 0 ? NB : 1];
                fval(f, q * Q + i);
                dp_place<NB, double>(st, f);
            }
        }
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int64_t x = x0 + q * Q + i;
            double f[NB > 0 ? NB : 1];
            fval(f, q * Q + i);
            dp_diag<NB, double, true>(F, wt);
            dp_place<NB, double>(F, f);
            const double J = combine<NB, double>(F, H[i]);
            if (x < N) {
                const double mu = muk[x];
                if (MODE == MODE_UPD) {
                    const double qv = div_nr1(mu, J);
                    const bool nz = nonzero(mu);
                    bad |= nz && !finite_positive(qv);
                    if (DEFER) {
                        acc += fabs(phik[x] * J - mu);
                        cp.scr[inst * N + x] = nz ? qv : 0.0;
                    } else {
                        phik[x] = nz ? qv : 0.0;
                    }
                } else {
                    acc += fabs(phik[x] * J - mu);
                }
            }
        }
    }
    __syncthreads();  // phi_k complete (UPD) / shared aggregates free for the next product
    return acc;
}

template <int NB, int P>
__global__ void __launch_bounds__(kCtaT, 1) k_cta_sinkhorn(CtaPlan cp) {
    constexpr int L = NB + 1, SZ = (NB + 1) << NB;
    __shared__ double aggF[kCtaW][SZ], aggB[kCtaW][SZ];
    __shared__ double red[kCtaW];
    const int64_t inst = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double wt[NB + 2];
    {
        const double eta = cp.eta[inst];
#pragma unroll
        for (int a = 0; a <= NB + 1; ++a) wt[a] = a <= L ? exp(-(double)(a * (L - a)) * cp.h / eta) : 0.0;
    }
    int done = 0, fail = -1;
    bool conv = false;
    double res = __longlong_as_double(0x7ff8000000000000ll);
    // block sum of one value per thread
    auto block_sum = [&](double a) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) red[w] = a;
        __syncthreads();
        double r = 0.0;
#pragma unroll
        for (int i = 0; i < kCtaW; ++i) r += red[i];
        __syncthreads();
        return r;
    };
    // Residual of a check sweep t < iters: the k = 0 term rides on sweep t+1's first update (its
    // bound vectors are sweep t's end-of-sweep ones), which writes phi_0 to scratch; if the total
    // meets tol the solve stops at sweep t and the scratch is dropped (l + l-2 products per check
    // sweep instead of l + l-1, as in the persistent kernel).
    bool pend = false;
    double pres = 0.0;
    int pt = 0;
    const int64_t x0 = (int64_t)threadIdx.x * P;
    for (int t = 1; t <= cp.iters; ++t) {
        bool bad = false;
        for (int k = 0; k < L; ++k) {
            if (k == 0 && pend) {
                const double r0 = block_sum(cta_product<NB, P, MODE_UPD, true>(cp, inst, 0, wt, aggF, aggB, bad));
                pend = false;
                res = pres + r0;
                if (res <= cp.tol && !__syncthreads_or(bad)) {
                    conv = true;
                    done = pt;
                    break;
                }
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if (x0 + j < cp.N) cp.phi[0][inst * cp.N + x0 + j] = cp.scr[inst * cp.N + x0 + j];
                __syncthreads();
            } else {
                cta_product<NB, P, MODE_UPD>(cp, inst, k, wt, aggF, aggB, bad);
            }
        }
        if (conv) break;
        if (__syncthreads_or(bad)) {
            fail = t;
            break;
        }
        done = t;
        if (cp.tol > 0 && (t % cp.check_every == 0 || t == cp.iters)) {
            // Res_t = sum_{k < l-1} ||phi_k J_k - mu_k||_1 on the end-of-sweep scalings
            const bool defer = t < cp.iters;
            double a = 0.0;
            for (int k = defer ? 1 : 0; k + 1 < L; ++k) a += cta_product<NB, P, MODE_RES>(cp, inst, k, wt, aggF, aggB, bad);
            const double r = block_sum(a);
            if (defer) {
                pend = true;
                pres = r;
                pt = t;
            } else {
                res = r;
                if (r <= cp.tol) {
                    conv = true;
                    break;
                }
            }
        }
    }
    if (threadIdx.x == 0) {
        cp.status[inst] = fail >= 0 ? 6 : 0;
        cp.fail_iter[inst] = fail;
        cp.iters_done[inst] = done;
        cp.converged[inst] = conv ? 1 : 0;
        cp.resid[inst] = res;
    }
}

// u (caller layout, LOG or LINEAR) <-> phi (linear fp64), op 0 import, 1 export
__global__ void k_cta_convert(CtaPlan cp, void *const *u, int op, int log_repr) {
    const int64_t n = cp.batch * cp.N;
    const int q = blockIdx.y;
    double *phi = cp.phi[q];
    double *uu = reinterpret_cast<double *const *>(u)[q];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (op == 0) phi[i] = log_repr ? exp(uu[i]) : uu[i];
        else uu[i] = log_repr ? log(phi[i]) : phi[i];
    }
}

cudaError_t launch_cta_convert(const CtaPlan &cp, void *const *u_dev, int op, int log_repr, cudaStream_t s,
                               int64_t *launches) {
    const int64_t n = cp.batch * cp.N;
    dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)cp.l);
    k_cta_convert<<<g, 256, 0, s>>>(cp, u_dev, op, log_repr);
    ++*launches;
    return cudaGetLastError();
}

int cta_chain_len(int64_t N) {
    int P = 1;
    while ((int64_t)P * kCtaT < N) P <<= 1;
    return P;
}

template <int NB>
static cudaError_t cta_go(const CtaPlan &cp, cudaStream_t s) {
    const unsigned g = (unsigned)cp.batch;
    switch (cp.P) {
        case 1: k_cta_sinkhorn<NB, 1><<<g, kCtaT, 0, s>>>(cp); break;
        case 2: k_cta_sinkhorn<NB, 2><<<g, kCtaT, 0, s>>>(cp); break;
        case 4: k_cta_sinkhorn<NB, 4><<<g, kCtaT, 0, s>>>(cp); break;
        case 8: k_cta_sinkhorn<NB, 8><<<g, kCtaT, 0, s>>>(cp); break;
        case 16: k_cta_sinkhorn<NB, 16><<<g, kCtaT, 0, s>>>(cp); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_cta_sinkhorn(const CtaPlan &cp, cudaStream_t s, int64_t *launches) {
    ++*launches;
    switch (cp.l - 1) {
        case 1: return cta_go<1>(cp, s);
        case 2: return cta_go<2>(cp, s);
        case 3: return cta_go<3>(cp, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mmot
