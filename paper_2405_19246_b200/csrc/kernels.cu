// kernels.cu -- v0 kernels of the O(N) tensor-vector product on sm_100a.
//
// One product J_k = three phases, all on device:
//   1. k_chunk_ops   : one thread per chunk of P grid points walks its chunk once left-to-
//                      right and once right-to-left and builds the chunk's prefix and
//                      suffix operators (the shifted DPs G_c of dp.cuh).
//   2. k_ops_reduce / k_ops_down : hierarchical scan of the operators (groups of 32) ->
//                      the exact prefix state F entering every chunk and the exact suffix
//                      state B leaving it (both directions in one launch, blockIdx.y).
//   3. k_chunk_apply : one thread per chunk re-walks its chunk with the true carries:
//                      suffix states are checkpointed every Q points (local memory), then
//                      for each Q-block the suffix states are rebuilt in registers and the
//                      prefix walk combines J[m] = sum_S F_m[S] (w_{|S|+1} B_{m+1})[S^c]
//                      and applies the epilogue of the mode (marginal / update / residual /
//                      cost).
// Everything is fp64 (double or dual numbers for the cost).
#include <cuda_runtime.h>
#include <math.h>

#include "internal.h"

namespace mmot {

// ---------------------------------------------------------------------------------------
template <int NB, typename T>
__device__ __forceinline__ void load_weights(T (&wt)[NB + 2], const Weights &W) {
#pragma unroll
    for (int a = 0; a <= NB + 1; ++a) load_weight(wt[a], W, a);
}

template <int NB>
__device__ __forceinline__ void load_f(double (&f)[NB > 0 ? NB : 1], const Plan &p, int64_t x) {
#pragma unroll
    for (int b = 0; b < NB; ++b) f[b] = __ldg(p.bound[b] + x);
}

// ---------------------------------------------------------------------------------------
// Phase 1: chunk operators.
// ---------------------------------------------------------------------------------------
template <int NB, typename T>
__global__ void __launch_bounds__(128) k_chunk_ops(Plan p) {
    constexpr int M = 1 << NB;
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= p.nchunks || *p.stop) return;
    const int64_t x0 = c * p.P;
    const int64_t x1 = min(p.N, x0 + p.P);
    T wt[NB + 2];
    load_weights<NB, T>(wt, p.W);
    T G[NB + 1][M];
    double f[NB > 0 ? NB : 1];
    op_identity<NB, T>(G);
    for (int64_t x = x0; x < x1; ++x) {
        load_f<NB>(f, p, x);
        op_step<NB, T>(G, wt, f);
    }
    op_store<NB, T>(G, static_cast<T *>(p.ops_f[0]) + c * OpShape<NB>::SZ);
    op_identity<NB, T>(G);
    for (int64_t x = x1 - 1; x >= x0; --x) {
        load_f<NB>(f, p, x);
        op_step<NB, T>(G, wt, f);
    }
    op_store<NB, T>(G, static_cast<T *>(p.ops_b[0]) + c * OpShape<NB>::SZ);
}

// ---------------------------------------------------------------------------------------
// Phase 2a: compose groups of kGroup consecutive operators (dir 0: prefix order, dir 1:
// suffix order, i.e. the last member is applied first).
// ---------------------------------------------------------------------------------------
template <int NB, typename T>
__global__ void __launch_bounds__(64) k_ops_reduce(const T *in_f, const T *in_b, T *out_f, T *out_b,
                                                   int64_t n_in, const int *stop) {
    constexpr int M = 1 << NB;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int dir = blockIdx.y;
    const int64_t first = g * kGroup;
    if (first >= n_in || *stop) return;
    const int64_t last = min(n_in, first + kGroup) - 1;
    const T *in = dir == 0 ? in_f : in_b;
    T *out = dir == 0 ? out_f : out_b;
    T A[NB + 1][M], B[NB + 1][M], C[NB + 1][M];
    if (dir == 0) {
        op_load<NB, T>(A, in + first * OpShape<NB>::SZ);
        for (int64_t i = first + 1; i <= last; ++i) {
            op_load<NB, T>(B, in + i * OpShape<NB>::SZ);
            op_compose<NB, T>(A, B, C);
#pragma unroll
            for (int cc = 0; cc <= NB; ++cc)
#pragma unroll
                for (int S = 0; S < M; ++S) A[cc][S] = C[cc][S];
        }
    } else {
        op_load<NB, T>(A, in + last * OpShape<NB>::SZ);
        for (int64_t i = last - 1; i >= first; --i) {
            op_load<NB, T>(B, in + i * OpShape<NB>::SZ);
            op_compose<NB, T>(A, B, C);
#pragma unroll
            for (int cc = 0; cc <= NB; ++cc)
#pragma unroll
                for (int S = 0; S < M; ++S) A[cc][S] = C[cc][S];
        }
    }
    op_store<NB, T>(A, out + g * OpShape<NB>::SZ);
}

// Phase 2b: starting from each group's carry (or the empty set for the top level), apply
// the member operators in order and record every member's carry-in.
template <int NB, typename T>
__global__ void __launch_bounds__(64) k_ops_down(const T *ops_f, const T *ops_b, const T *gcar_f,
                                                 const T *gcar_b, T *car_f, T *car_b, int64_t n_in,
                                                 const int *stop) {
    constexpr int M = 1 << NB;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int dir = blockIdx.y;
    const int64_t first = g * kGroup;
    if (first >= n_in || *stop) return;
    const int64_t last = min(n_in, first + kGroup) - 1;
    const T *ops = dir == 0 ? ops_f : ops_b;
    const T *gc = dir == 0 ? gcar_f : gcar_b;
    T *car = dir == 0 ? car_f : car_b;
    T cur[M], nxt[M], G[NB + 1][M];
    if (gc) vec_load<NB, T>(cur, gc + g * M);
    else vec_unit<NB, T>(cur);
    if (dir == 0) {
        for (int64_t i = first; i <= last; ++i) {
            vec_store<NB, T>(cur, car + i * M);
            if (i == last) break;
            op_load<NB, T>(G, ops + i * OpShape<NB>::SZ);
            op_apply<NB, T>(G, cur, nxt);
#pragma unroll
            for (int S = 0; S < M; ++S) cur[S] = nxt[S];
        }
    } else {
        for (int64_t i = last; i >= first; --i) {
            vec_store<NB, T>(cur, car + i * M);
            if (i == first) break;
            op_load<NB, T>(G, ops + i * OpShape<NB>::SZ);
            op_apply<NB, T>(G, cur, nxt);
#pragma unroll
            for (int S = 0; S < M; ++S) cur[S] = nxt[S];
        }
    }
}

// ---------------------------------------------------------------------------------------
// Phase 3: apply.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void raise_status(const Plan &p, int st) {
    if (atomicCAS(p.status, 0, st) == 0) *p.fail_iter = p.iter;
    *(volatile int *)p.stop = 1;
}

template <int NB, typename T, int MODE>
__global__ void __launch_bounds__(128) k_chunk_apply(Plan p) {
    constexpr int M = 1 << NB;
    constexpr int Q = sub_q(NB);
    constexpr int NSUB = nsub_max(NB);
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= p.nchunks || *p.stop) return;
    const int64_t x0 = c * p.P;
    const int64_t x1 = min(p.N, x0 + p.P);
    const int nsub = (int)((x1 - x0 + Q - 1) / Q);
    T wt[NB + 2];
    load_weights<NB, T>(wt, p.W);
    T F[M], st[M];
    vec_load<NB, T>(F, static_cast<const T *>(p.car_f[0]) + c * M);
    vec_load<NB, T>(st, static_cast<const T *>(p.car_b[0]) + c * M);
    double f[NB > 0 ? NB : 1];
    // suffix walk with checkpoints: ck[j] = B at the right boundary of sub-block j
    T ck[NSUB][M];
    {
        int j = nsub - 1;
#pragma unroll
        for (int S = 0; S < M; ++S) ck[j][S] = st[S];
        for (int64_t x = x1 - 1; x > x0; --x) {
            load_f<NB>(f, p, x);
            dp_diag<NB, T>(st, wt);
            dp_place<NB, T>(st, f);
            if (x == x0 + (int64_t)j * Q) {
                --j;
#pragma unroll
                for (int S = 0; S < M; ++S) ck[j][S] = st[S];
            }
        }
    }
    double acc = 0.0;
    for (int j = 0; j < nsub; ++j) {
        const int64_t s0 = x0 + (int64_t)j * Q;
        const int len = (int)min((int64_t)Q, x1 - s0);
        double fq[Q][NB > 0 ? NB : 1];
        T H[Q][M];
#pragma unroll
        for (int i = 0; i < Q; ++i)
            if (i < len) load_f<NB>(fq[i], p, s0 + i);
#pragma unroll
        for (int S = 0; S < M; ++S) st[S] = ck[j][S];
        // rebuild H_m = diag(w) B_{m+1} for m = s0+len-1 .. s0
#pragma unroll
        for (int i = Q - 1; i >= 0; --i) {
            if (i < len) {
                dp_diag<NB, T>(st, wt);
#pragma unroll
                for (int S = 0; S < M; ++S) H[i][S] = st[S];
                if (i > 0) dp_place<NB, T>(st, fq[i]);
            }
        }
        // prefix walk + combine + epilogue
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            if (i < len) {
                const int64_t m = s0 + i;
                dp_diag<NB, T>(F, wt);
                dp_place<NB, T>(F, fq[i]);
                T J = zero_of(T{});
#pragma unroll
                for (int S = 0; S < M; ++S) J = mad(F[S], H[i][(M - 1) ^ S], J);
                if (MODE == MODE_MARG) {
                    p.outk[m] = p.phik[m] * value_of(J);
                } else if (MODE == MODE_UPD) {
                    const double mu = p.muk[m];
                    const double jv = value_of(J);
                    double phi = 0.0;
                    if (mu != 0.0) {
                        phi = mu / jv;
                        if (!(jv > 0.0) || !isfinite(jv) || !isfinite(phi)) raise_status(p, 6 /*EOVERFLOW*/);
                    }
                    p.outk[m] = phi;
                } else if (MODE == MODE_RES) {
                    acc += fabs(p.phik[m] * value_of(J) - p.muk[m]);
                } else {  // MODE_COST
                    if constexpr (sizeof(T) == sizeof(Dual)) acc += p.phik[m] * reinterpret_cast<const Dual &>(J).d;
                }
            }
        }
    }
    if (MODE == MODE_RES || MODE == MODE_COST) p.partial[c] = acc;
}

// ---------------------------------------------------------------------------------------
template <int NB, typename T>
static cudaError_t product_nb(const Plan &p, int mode, cudaStream_t s, int64_t *launches, cudaEvent_t *ev) {
    const int tpb = 128;
    const int64_t nb = (p.nchunks + tpb - 1) / tpb;
    if (ev) cudaEventRecord(ev[0], s);
    k_chunk_ops<NB, T><<<(unsigned)nb, tpb, 0, s>>>(p);
    if (ev) cudaEventRecord(ev[1], s);
    ++*launches;
    // up-sweep
    for (int i = 0; i + 1 < p.nlev; ++i) {
        const int64_t ng = p.nlev_n[i + 1];
        dim3 grid((unsigned)((ng + 63) / 64), 2);
        k_ops_reduce<NB, T><<<grid, 64, 0, s>>>(static_cast<const T *>(p.ops_f[i]), static_cast<const T *>(p.ops_b[i]),
                                               static_cast<T *>(p.ops_f[i + 1]), static_cast<T *>(p.ops_b[i + 1]),
                                               p.nlev_n[i], p.stop);
        ++*launches;
    }
    // down-sweep
    for (int i = p.nlev - 1; i >= 0; --i) {
        const int64_t ng = (p.nlev_n[i] + kGroup - 1) / kGroup;
        dim3 grid((unsigned)((ng + 63) / 64), 2);
        const T *gf = i + 1 < p.nlev ? static_cast<const T *>(p.car_f[i + 1]) : nullptr;
        const T *gb = i + 1 < p.nlev ? static_cast<const T *>(p.car_b[i + 1]) : nullptr;
        k_ops_down<NB, T><<<grid, 64, 0, s>>>(static_cast<const T *>(p.ops_f[i]), static_cast<const T *>(p.ops_b[i]),
                                             gf, gb, static_cast<T *>(p.car_f[i]), static_cast<T *>(p.car_b[i]),
                                             p.nlev_n[i], p.stop);
        ++*launches;
    }
    if (ev) cudaEventRecord(ev[2], s);
    switch (mode) {
        case MODE_MARG: k_chunk_apply<NB, T, MODE_MARG><<<(unsigned)nb, tpb, 0, s>>>(p); break;
        case MODE_UPD: k_chunk_apply<NB, T, MODE_UPD><<<(unsigned)nb, tpb, 0, s>>>(p); break;
        case MODE_RES: k_chunk_apply<NB, T, MODE_RES><<<(unsigned)nb, tpb, 0, s>>>(p); break;
        default: k_chunk_apply<NB, T, MODE_COST><<<(unsigned)nb, tpb, 0, s>>>(p); break;
    }
    ++*launches;
    if (ev) cudaEventRecord(ev[3], s);
    return cudaGetLastError();
}

cudaError_t launch_product(const Plan &p, int mode, cudaStream_t s, int64_t *launches, cudaEvent_t *ev) {
    const bool dual = mode == MODE_COST;
    switch (p.NB) {
        case 1: return dual ? product_nb<1, Dual>(p, mode, s, launches, ev) : product_nb<1, double>(p, mode, s, launches, ev);
        case 2: return dual ? product_nb<2, Dual>(p, mode, s, launches, ev) : product_nb<2, double>(p, mode, s, launches, ev);
        case 3: return dual ? product_nb<3, Dual>(p, mode, s, launches, ev) : product_nb<3, double>(p, mode, s, launches, ev);
        case 4: return dual ? product_nb<4, Dual>(p, mode, s, launches, ev) : product_nb<4, double>(p, mode, s, launches, ev);
        case 5: return dual ? product_nb<5, Dual>(p, mode, s, launches, ev) : product_nb<5, double>(p, mode, s, launches, ev);
        default: return cudaErrorInvalidValue;
    }
}

// ---------------------------------------------------------------------------------------
// Small kernels.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_sum(const double *partial, int64_t n, double *out, double scale,
                                              int accumulate, const int *stop) {
    __shared__ double sh[1024];
    if (*stop) return;
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += partial[i];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = (accumulate ? *out : 0.0) + scale * sh[0];
}

cudaError_t launch_sum(const double *partial, int64_t n, double *out, double scale, int accumulate,
                       const int *stop, cudaStream_t s, int64_t *launches) {
    k_sum<<<1, 1024, 0, s>>>(partial, n, out, scale, accumulate, stop);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_exp(const double *in, double *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = exp(in[i]);
}
__global__ void k_log(const double *in, double *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = log(in[i]);
}
__global__ void k_fill(double *out, double v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v;
}

static unsigned grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (unsigned)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

cudaError_t launch_exp(const double *in, double *out, int64_t n, cudaStream_t s, int64_t *launches) {
    k_exp<<<grid_for(n), 256, 0, s>>>(in, out, n);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_log(const double *in, double *out, int64_t n, cudaStream_t s, int64_t *launches) {
    k_log<<<grid_for(n), 256, 0, s>>>(in, out, n);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_fill(double *out, double v, int64_t n, cudaStream_t s, int64_t *launches) {
    k_fill<<<grid_for(n), 256, 0, s>>>(out, v, n);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_check(const double *v, int64_t n, int allow_neg_inf, int *flags, double *mass) {
    __shared__ double sh[256];
    int fl = 0;
    double a = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = v[i];
        if (isnan(x) || (isinf(x) && !(allow_neg_inf && x < 0))) fl |= 1;
        else if (x < 0 && !allow_neg_inf) fl |= 2;
        else if (!allow_neg_inf) a += x;
    }
    if (fl) atomicOr(flags, fl);
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0 && mass) atomicAdd(mass, sh[0]);
}

cudaError_t launch_check(const double *v, int64_t n, int allow_neg_inf, int *flags, double *mass,
                         cudaStream_t s, int64_t *launches) {
    k_check<<<grid_for(n), 256, 0, s>>>(v, n, allow_neg_inf, flags, mass);
    ++*launches;
    return cudaGetLastError();
}

// flags[0..nvec) per vector; mass[0..nmarg) per marginal.
__global__ void k_check_finish(const int *flags, const double *mass, int nvec, int nmarg, int *status, int *stop,
                               int *fail_iter) {
    int st = 0;
    for (int i = 0; i < nvec && !st; ++i) {
        if (flags[i] & 1) st = 3;       // ENONFINITE
        else if (flags[i] & 2) st = 4;  // ENEGMASS
    }
    for (int i = 0; i < nmarg && !st; ++i)
        if (!(mass[i] > 0.0)) st = 5;   // EZEROMASS
    if (st) {
        *status = st;
        *fail_iter = 0;
        *stop = 1;
    }
}

cudaError_t launch_check_finish(const int *flags, const double *mass, int nvec, int nmarg, int *status, int *stop,
                                int *fail_iter, cudaStream_t s, int64_t *launches) {
    k_check_finish<<<1, 1, 0, s>>>(flags, mass, nvec, nmarg, status, stop, fail_iter);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_resid_finish(double *acc, double tol, int iter, double *res_out, int *iters_done, int *converged,
                               int *stop) {
    if (*stop) return;
    const double r = *acc;
    *res_out = r;
    *iters_done = iter;
    if (r <= tol) {
        *converged = 1;
        *stop = 1;
    }
}

cudaError_t launch_resid_finish(double *acc, double tol, int iter, double *res_out, int *iters_done, int *converged,
                                int *stop, cudaStream_t s, int64_t *launches) {
    k_resid_finish<<<1, 1, 0, s>>>(acc, tol, iter, res_out, iters_done, converged, stop);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_sweep_done(int iter, int *iters_done, const int *stop) {
    if (!*stop) *iters_done = iter;
}

cudaError_t launch_sweep_done(int iter, int *iters_done, const int *stop, cudaStream_t s, int64_t *launches) {
    k_sweep_done<<<1, 1, 0, s>>>(iter, iters_done, stop);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace mmot
