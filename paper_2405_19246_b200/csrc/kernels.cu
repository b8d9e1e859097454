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
#include <algorithm>
#include <math.h>
#include <stdlib.h>

#include <mutex>
#include <set>
#include <tuple>

#include "internal.h"
#include "walk.cuh"

namespace mmot {

// MMOT_NO_TMEM=1 disables the TMEM checkpoint kernels (A/B testing).
static const bool g_no_tmem = [] { const char *e = getenv("MMOT_NO_TMEM"); return e && e[0] == '1'; }();

// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// Phase 1: chain operators (prefix walk and suffix walk of every chain).
// ---------------------------------------------------------------------------------------
constexpr int kWarpsPerCta = 4;

// Non-uniform grids: weights of grid edge e (between points e-1 and e) from the context's arrays.
template <int NB, typename T>
__device__ __forceinline__ void pweights_plan(T (&w)[NB + 2], const Plan &p, int64_t e) {
    pweights_val<NB, T>(w, __ldg(p.lam + e), sizeof(T) == sizeof(double) ? 0.0 : __ldg(p.hx + e));
}
// dp_diag with the uniform weights, or those of edge e on a non-uniform grid
template <int NB, typename T, bool PTS>
__device__ __forceinline__ void diag_e(T (&st)[1 << NB], const T (&wt)[NB + 2], const Plan &p, int64_t e) {
    if constexpr (PTS) {
        T w[NB + 2];
        pweights_plan<NB, T>(w, p, e);
        dp_diag<NB, T, true>(st, w);
    } else {
        dp_diag<NB, T, true>(st, wt);
    }
}

template <int NB, typename T, bool PTS = false, bool ALL = false>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_chunk_ops(Plan p) {
    constexpr int M = 1 << NB;
    constexpr int S = slab_s(NB);
    constexpr int TILE = 32 * (S + 1);
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t chain0 = ((int64_t)blockIdx.x * kWarpsPerCta + warp) * 32;
    if (chain0 >= p.nchunks || *p.stop) return;
    double *buf = smem + (size_t)warp * 2 * NB * TILE;
    const int64_t c = chain0 + lane;
    const int64_t x0 = c * p.P;
    const int64_t x1 = min(p.N, x0 + p.P);
    const int ns = (int)((p.P + S - 1) / S);
    T wt[NB + 2];
    load_weights<NB, T>(wt, p.W);
    T G[NB + 1][M];
    double f[NB > 0 ? NB : 1];
    // one left-to-right walk of the extended operator; prefix and suffix operators follow from
    // the duality R_c[V] = w_c Gt_{l-c-|V|}[V] (dp.cuh, opx_*)
    opx_identity<NB, T>(G);
    slab_issue<S, NB>(buf, p.bound, chain0, p.P, p.N, 0, lane);
    cp_async_commit();
    for (int s = 0; s < ns; ++s) {
        if (s + 1 < ns) slab_issue<S, NB>(buf + ((s + 1) & 1) * NB * TILE, p.bound, chain0, p.P, p.N, s + 1, lane);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const double *cur = buf + (s & 1) * NB * TILE;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const int64_t x = x0 + (int64_t)s * S + j;
            if (x < x1) {
                slab_f<NB, S>(f, cur, lane, j);
                if constexpr (PTS) {
                    T wx[NB + 2];
                    pweights_plan<NB, T>(wx, p, x);  // edge into point x
                    opx_step<NB, T>(G, wx, f, s == 0 && j == 0);
                } else {
                    opx_step<NB, T>(G, wt, f, s == 0 && j == 0);
                }
            }
        }
        __syncwarp();
    }
    if (c < p.nchunks) {
        if constexpr (PTS) {
            T win[NB + 2], wout[NB + 2];
            pweights_plan<NB, T>(win, p, x0);           // entry edge of the chunk
            pweights_plan<NB, T>(wout, p, x0 + p.P);    // exit edge (1 beyond the grid)
            opx_store_pts<NB, T>(G, win, wout, static_cast<T *>(p.ops_f[0]) + c * OpShape<NB>::SZ,
                                 static_cast<T *>(p.ops_b[0]) + c * OpShape<NB>::SZ);
        } else {
            opx_store<NB, T, ALL ? NB : NB + 1>(G, wt, static_cast<T *>(p.ops_f[0]) + c * OpShape<NB>::SZ,
                                                static_cast<T *>(p.ops_b[0]) + c * OpShape<NB>::SZ);
        }
    }
}

// k_chunk_ops for NB = 5 (fp64, uniform grid) split by operator slice: the extended walk's slices
// c = 0..NB never mix (diag scales G[c][V] by w_{c+|V|}, place stays inside slice c), so two
// threads per chunk walk slices {0,1,2} and {3,4,5} (96 doubles each instead of 192, which spill);
// the slices meet in shared memory for the store (the suffix operator reads slice l-c-|V|).
constexpr int kOpsSplitChunks = 32;  // chunks per block (64 threads)
template <int NB, bool ALL = false>
__global__ void __launch_bounds__(2 * kOpsSplitChunks) k_chunk_ops_split(Plan p) {
    constexpr int M = 1 << NB;
    constexpr int L = NB + 1;
    constexpr int HS = (NB + 1) / 2;  // slices per thread
    __shared__ double Gs[kOpsSplitChunks][NB + 1][M];
    const int ci = threadIdx.x >> 1, half = threadIdx.x & 1;
    const int64_t c = (int64_t)blockIdx.x * kOpsSplitChunks + ci;
    if (*p.stop) return;
    double wt[NB + 2];
    load_weights<NB, double>(wt, p.W);
    double G[HS][M];
#pragma unroll
    for (int i = 0; i < HS; ++i)
#pragma unroll
        for (int V = 0; V < M; ++V) G[i][V] = V == 0 ? 1.0 : 0.0;
    if (c < p.nchunks) {
        const int64_t x0 = c * p.P, x1 = min(p.N, x0 + p.P);
        for (int64_t x = x0; x < x1; ++x) {
            double f[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = __ldg(p.bound[b] + x);
            const bool skip = x == x0;
#pragma unroll
            for (int i = 0; i < HS; ++i) {
                const int cc = half * HS + i;
                if (!skip) {
#pragma unroll
                    for (int V = 0; V < M; ++V) {
                        const int a = cc + pc(V);
                        if (a < L && a > 0) G[i][V] *= wt[a];
                    }
                }
#pragma unroll
                for (int b = 0; b < NB; ++b)
#pragma unroll
                    for (int V = M - 1; V >= 0; --V)
                        if (((V >> b) & 1) && cc + pc(V) <= L) G[i][V] = fma(f[b], G[i][V ^ (1 << b)], G[i][V]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < HS; ++i)
#pragma unroll
        for (int V = 0; V < M; ++V) Gs[ci][half * HS + i][V] = G[i][V];
    __syncthreads();
    if (c >= p.nchunks) return;
    double *pf = static_cast<double *>(p.ops_f[0]) + c * OpShape<NB>::SZ;
    double *pb = static_cast<double *>(p.ops_b[0]) + c * OpShape<NB>::SZ;
    // opx_store: prefix w_c Gt_c, suffix w_c Gt_{l-c-|V|} (this thread: slices half*HS ..)
#pragma unroll
    for (int i = 0; i < HS; ++i) {
        const int cc = half * HS + i;
#pragma unroll
        for (int V = 0; V < M; ++V)
            if (cc + pc(V) <= NB) {
                const int cp = (ALL ? NB : NB + 1) - cc - pc(V);
                pf[cc * M + V] = cc == 0 ? Gs[ci][0][V] : wt[cc] * Gs[ci][cc][V];
                const double r = cp > NB ? 1.0 : Gs[ci][cp][V];
                pb[cc * M + V] = cc == 0 ? r : wt[cc] * r;
            }
    }
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
    const int64_t first = g * group_of(NB);
    if (first >= n_in || *stop) return;
    const int64_t last = min(n_in, first + group_of(NB)) - 1;
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
                                                 const int *stop, T *car_bi) {
    constexpr int M = 1 << NB;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int dir = blockIdx.y;
    const int64_t first = g * group_of(NB);
    if (first >= n_in || *stop) return;
    const int64_t last = min(n_in, first + group_of(NB)) - 1;
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
            if (i == first && !car_bi) break;
            op_load<NB, T>(G, ops + i * OpShape<NB>::SZ);
            op_apply<NB, T>(G, cur, nxt);
#pragma unroll
            for (int S = 0; S < M; ++S) cur[S] = nxt[S];
            if (car_bi) vec_store<NB, T>(cur, car_bi + i * M);  // inclusive: suffix state at chain start
        }
    }
}

// Block-cooperative variants of phase 2 for large operators (NB >= 4): a group of group_of(NB)
// operators is staged in shared memory and every output entry (c, V) of a composition / every
// state of an application is computed by its own thread, so the serial chain per group is
// log2(group) compositions (reduce) or group applications of depth one (down).
template <int NB>
__device__ __forceinline__ bool opx_valid(int e) {  // entry e = c*M + V is a used operator entry
    constexpr int M = 1 << NB;
    return pc(e % M) <= NB - e / M;
}

// Term table of one composition C_c[V] = sum_{U subset V} X_c[U] Y_{c+|U|}[V\U] (NB >= 4): for
// output entry q = c*M + V the terms start[q] .. start[q+1]-1, each a packed pair of offsets
// (X offset | Y offset << 16) -- generated at compile time, staged in shared memory, so the
// reduce kernel spends two loads and one FMA per term instead of the subset-enumeration
// arithmetic.
template <int NB>
struct ComposeTab {
    static constexpr int M = 1 << NB;
    static constexpr int SZ = (NB + 1) * M;
    static constexpr int count_terms() {
        int n = 0;
        for (int q = 0; q < SZ; ++q) {
            const int c = q / M, V = q % M;
            if (pc(V) <= NB - c) n += 1 << pc(V);
        }
        return n;
    }
    static constexpr int NT = count_terms();
    unsigned pair[NT];
    unsigned short start[SZ + 1];
    constexpr ComposeTab() : pair(), start() {
        int n = 0;
        for (int q = 0; q < SZ; ++q) {
            start[q] = (unsigned short)n;
            const int c = q / M, V = q % M;
            if (pc(V) > NB - c) continue;
            int U = V;
            for (int t = 0; t < (1 << pc(V)); ++t) {
                pair[n++] = (unsigned)(c * M + U) | ((unsigned)((c + pc(U)) * M + (V ^ U)) << 16);
                U = (U - 1) & V;
            }
        }
        start[SZ] = (unsigned short)n;
    }
};
template <int NB>
__device__ const ComposeTab<NB> g_ctab = ComposeTab<NB>();

// fp64 reduce for NB >= 4 through the term table (layout and semantics as k_ops_reduce_c).
template <int NB>
__global__ void __launch_bounds__(128) k_ops_reduce_t(const double *in_f, const double *in_b, double *out_f,
                                                     double *out_b, int64_t n_in, const int *stop) {
    constexpr int M = 1 << NB;
    constexpr int SZ = OpShape<NB>::SZ;
    constexpr int GS = group_of(NB);
    constexpr int NT = ComposeTab<NB>::NT;
    __shared__ double A[GS][SZ];
    __shared__ unsigned tp[NT];
    __shared__ unsigned short ts[SZ + 1];
    const int64_t g = blockIdx.x;
    const int dir = blockIdx.y;
    const int64_t first = g * GS;
    if (first >= n_in || *stop) return;
    for (int t = threadIdx.x; t < NT; t += blockDim.x) tp[t] = g_ctab<NB>.pair[t];
    for (int t = threadIdx.x; t <= SZ; t += blockDim.x) ts[t] = g_ctab<NB>.start[t];
    const int cnt = (int)min((int64_t)GS, n_in - first);
    const double *in = (dir == 0 ? in_f : in_b) + first * SZ;
    for (int e = threadIdx.x; e < GS * SZ; e += blockDim.x) {
        const int i = e / SZ, q = e % SZ;
        A[i][q] = i < cnt && opx_valid<NB>(q) ? in[e] : ((q % M) == 0 && i >= cnt ? 1.0 : 0.0);
    }
    __syncthreads();
    constexpr int IT = (GS / 2 * SZ + 127) / 128;
#pragma unroll
    for (int step = 1; step < GS; step <<= 1) {
        const int lim = (GS / (2 * step)) * SZ;
        double res[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * 128;
            res[it] = 0.0;
            if (e < lim) {
                const int pr = e / SZ, q = e % SZ;
                const int i = pr * 2 * step;
                const double *X = dir == 0 ? A[i] : A[i + step];  // applied first
                const double *Y = dir == 0 ? A[i + step] : A[i];  // applied second
                double a0 = 0.0, a1 = 0.0;
                const int t0 = ts[q], t1 = ts[q + 1];
                int t = t0;
#pragma unroll 2
                for (; t + 1 < t1; t += 2) {
                    const unsigned p0 = tp[t], p1 = tp[t + 1];
                    a0 = fma(X[p0 & 0xffffu], Y[p0 >> 16], a0);
                    a1 = fma(X[p1 & 0xffffu], Y[p1 >> 16], a1);
                }
                if (t < t1) {
                    const unsigned p0 = tp[t];
                    a0 = fma(X[p0 & 0xffffu], Y[p0 >> 16], a0);
                }
                res[it] = a0 + a1;
            }
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * 128;
            if (e < lim) A[(e / SZ) * 2 * step][e % SZ] = res[it];
        }
        __syncthreads();
    }
    double *out = (dir == 0 ? out_f : out_b) + g * SZ;
    for (int q = threadIdx.x; q < SZ; q += blockDim.x)
        if (opx_valid<NB>(q)) out[q] = A[0][q];
}

template <int NB, typename T>
__global__ void __launch_bounds__(128) k_ops_reduce_c(const T *in_f, const T *in_b, T *out_f, T *out_b, int64_t n_in,
                                                       const int *stop) {
    constexpr int M = 1 << NB;
    constexpr int SZ = OpShape<NB>::SZ;
    constexpr int GS = group_of(NB);
    __shared__ T A[GS][SZ];
    const int64_t g = blockIdx.x;
    const int dir = blockIdx.y;
    const int64_t first = g * GS;
    if (first >= n_in || *stop) return;
    const int cnt = (int)min((int64_t)GS, n_in - first);
    const T *in = (dir == 0 ? in_f : in_b) + first * SZ;
    for (int e = threadIdx.x; e < GS * SZ; e += blockDim.x) {
        const int i = e / SZ, q = e % SZ;
        A[i][q] = i < cnt && opx_valid<NB>(q) ? in[e] : ((q % M) == 0 && i >= cnt ? one_of(T{}) : zero_of(T{}));
    }
    __syncthreads();
    constexpr int IT = (GS / 2 * SZ + 127) / 128;  // entries per thread at the widest step
#pragma unroll
    for (int step = 1; step < GS; step <<= 1) {
        // pairs (i, i + step), i a multiple of 2 step; prefix order applies member i first,
        // suffix order applies member i + step first
        const int lim = (GS / (2 * step)) * SZ;
        T res[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * 128;
            res[it] = zero_of(T{});
            if (e < lim) {
                const int pr = e / SZ, q = e % SZ;
                const int c = q / M, V = q % M;
                const int i = pr * 2 * step;
                const T *X = dir == 0 ? A[i] : A[i + step];      // applied first
                const T *Y = dir == 0 ? A[i + step] : A[i];      // applied second
                if (pc(V) <= NB - c) {
                    // C_c[V] = sum_{U subset V} X_c[U] Y_{c+|U|}[V\U]: 2^|V| terms, counted loop
                    // (two accumulators, unrolled so the shared-memory loads run ahead)
                    const int nt = 1 << pc(V);
                    T a0 = zero_of(T{}), a1 = zero_of(T{});
                    int U = V;
#pragma unroll 4
                    for (int t = 0; t < nt; ++t) {
                        const T x = X[c * M + U], y = Y[(c + pc(U)) * M + (V ^ U)];
                        if (t & 1) a1 = mad(x, y, a1);
                        else a0 = mad(x, y, a0);
                        U = (U - 1) & V;
                    }
                    res[it] = a0 + a1;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int e = threadIdx.x + it * 128;
            if (e < lim) A[(e / SZ) * 2 * step][e % SZ] = res[it];
        }
        __syncthreads();
    }
    T *out = (dir == 0 ? out_f : out_b) + g * SZ;
    for (int q = threadIdx.x; q < SZ; q += blockDim.x)
        if (opx_valid<NB>(q)) out[q] = A[0][q];
}

template <int NB, typename T>
__global__ void __launch_bounds__(64) k_ops_down_c(const T *ops_f, const T *ops_b, const T *gcar_f, const T *gcar_b,
                                                    T *car_f, T *car_b, int64_t n_in, const int *stop, T *car_bi) {
    constexpr int M = 1 << NB;
    constexpr int SZ = OpShape<NB>::SZ;
    constexpr int GS = group_of(NB);
    __shared__ T G[GS][SZ];
    __shared__ T cur[M];
    const int64_t g = blockIdx.x;
    const int dir = blockIdx.y;
    const int64_t first = g * GS;
    if (first >= n_in || *stop) return;
    const int cnt = (int)min((int64_t)GS, n_in - first);
    const T *ops = (dir == 0 ? ops_f : ops_b) + first * SZ;
    for (int e = threadIdx.x; e < cnt * SZ; e += blockDim.x) G[e / SZ][e % SZ] = opx_valid<NB>(e % SZ) ? ops[e] : zero_of(T{});
    const T *gc = dir == 0 ? gcar_f : gcar_b;
    for (int S = threadIdx.x; S < M; S += blockDim.x) cur[S] = gc ? gc[g * M + S] : (S == 0 ? one_of(T{}) : zero_of(T{}));
    __syncthreads();
    T *car = dir == 0 ? car_f : car_b;
    for (int t = 0; t < cnt; ++t) {
        const int i = dir == 0 ? t : cnt - 1 - t;
        T nx = zero_of(T{});
        const int S = threadIdx.x;
        if (S < M) {
            car[(first + i) * M + S] = cur[S];
            // Op(cur)[S] = sum_{U subset S} cur[U] G_|U|[S\U]
            const int nt = 1 << pc(S);
            T a0 = zero_of(T{}), a1 = zero_of(T{});
            int U = S;
#pragma unroll 4
            for (int t = 0; t < nt; ++t) {
                const T x = cur[U], y = G[i][pc(U) * M + (S ^ U)];
                if (t & 1) a1 = mad(x, y, a1);
                else a0 = mad(x, y, a0);
                U = (U - 1) & S;
            }
            nx = a0 + a1;
        }
        __syncthreads();
        if (S < M) {
            cur[S] = nx;
            if (dir == 1 && car_bi) car_bi[(first + i) * M + S] = nx;  // inclusive (chain start)
        }
        __syncthreads();
    }
}

// Warp-per-group down-sweep for NB >= 4 (fp64): the M <= 32 states of an application map onto the
// lanes of one warp, so the group's GS sequential applications need only warp barriers; two
// groups per 64-thread block (blockIdx.y = direction as in k_ops_down_c).
template <int NB>
__global__ void __launch_bounds__(64) k_ops_down_cw(const double *ops_f, const double *ops_b, const double *gcar_f,
                                                     const double *gcar_b, double *car_f, double *car_b, int64_t n_in,
                                                     const int *stop, double *car_bi) {
    constexpr int M = 1 << NB;
    constexpr int SZ = OpShape<NB>::SZ;
    constexpr int GS = group_of(NB);
    __shared__ double G[2][GS][SZ];
    __shared__ double cur[2][M];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t g = (int64_t)blockIdx.x * 2 + w;
    const int dir = blockIdx.y;
    const int64_t first = g * GS;
    if (first >= n_in || *stop) return;
    const int cnt = (int)min((int64_t)GS, n_in - first);
    const double *ops = (dir == 0 ? ops_f : ops_b) + first * SZ;
    for (int e = lane; e < cnt * SZ; e += 32) G[w][e / SZ][e % SZ] = opx_valid<NB>(e % SZ) ? ops[e] : 0.0;
    const double *gc = dir == 0 ? gcar_f : gcar_b;
    if (lane < M) cur[w][lane] = gc ? gc[g * M + lane] : (lane == 0 ? 1.0 : 0.0);
    __syncwarp();
    double *car = dir == 0 ? car_f : car_b;
    for (int t = 0; t < cnt; ++t) {
        const int i = dir == 0 ? t : cnt - 1 - t;
        double nx = 0.0;
        if (lane < M) {
            car[(first + i) * M + lane] = cur[w][lane];
            // Op(cur)[S] = sum_{U subset S} cur[U] G_|U|[S\U]
            const int nt = 1 << pc(lane);
            double a0 = 0.0, a1 = 0.0;
            int U = lane;
#pragma unroll 4
            for (int k = 0; k < nt; ++k) {
                const double x = cur[w][U], y = G[w][i][pc(U) * M + (lane ^ U)];
                if (k & 1) a1 = fma(x, y, a1);
                else a0 = fma(x, y, a0);
                U = (U - 1) & lane;
            }
            nx = a0 + a1;
        }
        __syncwarp();
        if (lane < M) {
            cur[w][lane] = nx;
            if (dir == 1 && car_bi) car_bi[(first + i) * M + lane] = nx;  // inclusive (chain start)
        }
        __syncwarp();
    }
}

// Warp-cooperative variants of phase 2 (fp64, NB <= 3): one warp per group of 32 operators;
// the group is staged through shared memory (coalesced), then composed with a shuffle tree
// (reduce) or a Kogge-Stone scan (down).  blockIdx.y selects the direction.
template <int NB>
__device__ __forceinline__ void op_shfl(double (&dst)[NB + 1][1 << NB], const double (&src)[NB + 1][1 << NB],
                                        int delta, int mode /*0 idx, 1 up, 2 down*/) {
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int S = 0; S < (1 << NB); ++S) {
            if (pc(S) > NB - c) { dst[c][S] = 0.0; continue; }
            dst[c][S] = mode == 1 ? __shfl_up_sync(0xffffffffu, src[c][S], delta)
                                  : (mode == 2 ? __shfl_down_sync(0xffffffffu, src[c][S], delta)
                                               : __shfl_sync(0xffffffffu, src[c][S], delta));
        }
}

template <int NB>
__device__ __forceinline__ void op_stage_load(double (&G)[NB + 1][1 << NB], double *sm, const double *src, int64_t first,
                                              int64_t n_in, int lane) {
    constexpr int SZ = OpShape<NB>::SZ;
    const int64_t avail = min((int64_t)32, n_in - first);
    for (int e = lane; e < 32 * SZ; e += 32) {
        const int r = e / SZ, q = e % SZ;
        sm[r * (SZ + 1) + q] = r < avail ? src[first * SZ + e] : (q == 0 || q % (1 << NB) == 0 ? 1.0 : 0.0);
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int S = 0; S < (1 << NB); ++S)
            G[c][S] = pc(S) <= NB - c ? sm[lane * (SZ + 1) + c * (1 << NB) + S] : 0.0;
    __syncwarp();
}

template <int NB>
__global__ void __launch_bounds__(128) k_ops_reduce_w(const double *in_f, const double *in_b, double *out_f,
                                                     double *out_b, int64_t n_in, const int *stop) {
    constexpr int M = 1 << NB;
    constexpr int SZ = OpShape<NB>::SZ;
    __shared__ double smem[4][32 * (SZ + 1)];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t g = (int64_t)blockIdx.x * 4 + warp;
    const int dir = blockIdx.y;
    const int64_t first = g * kGroup;
    if (first >= n_in || *stop) return;
    double A[NB + 1][M], B[NB + 1][M], C[NB + 1][M];
    op_stage_load<NB>(A, smem[warp], dir == 0 ? in_f : in_b, first, n_in, lane);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        op_shfl<NB>(B, A, d, 2);
        if (dir == 0) op_compose<NB, double>(A, B, C);
        else op_compose<NB, double>(B, A, C);
        if ((lane & (2 * d - 1)) == 0) {
#pragma unroll
            for (int cc = 0; cc <= NB; ++cc)
#pragma unroll
                for (int S = 0; S < M; ++S) A[cc][S] = C[cc][S];
        }
    }
    if (lane == 0) op_store<NB, double>(A, (dir == 0 ? out_f : out_b) + g * SZ);
}

template <int NB>
__global__ void __launch_bounds__(128) k_ops_down_w(const double *ops_f, const double *ops_b, const double *gcar_f,
                                                   const double *gcar_b, double *car_f, double *car_b, int64_t n_in,
                                                   const int *stop, double *car_bi) {
    constexpr int M = 1 << NB;
    constexpr int SZ = OpShape<NB>::SZ;
    __shared__ double smem[4][32 * (SZ + 1)];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t g = (int64_t)blockIdx.x * 4 + warp;
    const int dir = blockIdx.y;
    const int64_t first = g * kGroup;
    if (first >= n_in || *stop) return;
    double A[NB + 1][M], B[NB + 1][M], C[NB + 1][M];
    op_stage_load<NB>(A, smem[warp], dir == 0 ? ops_f : ops_b, first, n_in, lane);
    // inclusive Kogge-Stone scan of the member operators in application order
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        op_shfl<NB>(B, A, d, dir == 0 ? 1 : 2);
        op_compose<NB, double>(B, A, C);  // the earlier-applied prefix B first, then A
        const bool take = dir == 0 ? lane >= d : lane + d < 32;
        if (take) {
#pragma unroll
            for (int cc = 0; cc <= NB; ++cc)
#pragma unroll
                for (int S = 0; S < M; ++S) A[cc][S] = C[cc][S];
        }
    }
    const double *gc = dir == 0 ? gcar_f : gcar_b;
    double cin[M], out[M], nb[M];
    if (gc) vec_load<NB, double>(cin, gc + g * M);
    else vec_unit<NB, double>(cin);
    op_apply<NB, double>(A, cin, out);
#pragma unroll
    for (int S = 0; S < M; ++S)
        nb[S] = dir == 0 ? __shfl_up_sync(0xffffffffu, out[S], 1) : __shfl_down_sync(0xffffffffu, out[S], 1);
    const bool edge = dir == 0 ? lane == 0 : lane == 31;
    const int64_t i = first + lane;
    if (i < n_in) {
        double *dst = (dir == 0 ? car_f : car_b) + i * M;
#pragma unroll
        for (int S = 0; S < M; ++S) dst[S] = edge ? cin[S] : nb[S];
        if (dir == 1 && car_bi) {
#pragma unroll
            for (int S = 0; S < M; ++S) car_bi[i * M + S] = out[S];  // inclusive: suffix state at chain start
        }
    }
}

// ---------------------------------------------------------------------------------------
// Phase 3: apply.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void raise_status(const Plan &p, int st) {
    // fail_iter: the sweep in progress (completed sweeps + 1 inside a solve; p.iter otherwise)
    if (atomicCAS(p.status, 0, st) == 0) *p.fail_iter = p.sweep ? *p.sweep + 1 : p.iter;
    *(volatile int *)p.stop = 1;
}

// Vectors staged by the apply phase: the NB bound vectors, then mu_k (update / residual),
// then phi_k (marginal / residual / cost).
// MODE_ALLRES: the NB = l scalings, then mu_0 .. mu_{l-2}.
template <int NB, int MODE>
struct ApplyVecs {
    static constexpr bool kMu = MODE == MODE_UPD || MODE == MODE_RES;
    static constexpr bool kPhi = MODE == MODE_MARG || MODE == MODE_RES || MODE == MODE_COST;
    static constexpr int NV = MODE == MODE_ALLRES ? 2 * NB - 1 : NB + (kMu ? 1 : 0) + (kPhi ? 1 : 0);
    static constexpr int IMU = NB;
    static constexpr int IPHI = NB + (kMu ? 1 : 0);
    static constexpr bool kOut = MODE == MODE_MARG || MODE == MODE_UPD;
};

// ---------------------------------------------------------------------------------------
// Tensor memory (TMEM) as a per-warp checkpoint store.  The path has no MMA, so the 256 KB of
// TMEM per SM are free; a CTA of 4 warps allocates 256 columns (2 CTAs per SM), warp w owns TMEM
// lanes [32w, 32w+32) and therefore 256 x 32-bit words per lane: 128 doubles = the suffix
// checkpoints of one chain (every 2Q points), instead of local memory that spills to DRAM.
// ---------------------------------------------------------------------------------------
constexpr int kTmemCols = 256;

__device__ __forceinline__ void tmem_alloc(uint32_t *smem_slot) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem_slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(a), "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(kTmemCols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// Store / load M doubles (2M 32-bit columns) of this thread's TMEM lane at column offset col.
template <int M>
__device__ __forceinline__ void tmem_st_vec(uint32_t taddr, const double (&v)[M]) {
    uint32_t r[2 * M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        r[2 * i] = __double2loint(v[i]);
        r[2 * i + 1] = __double2hiint(v[i]);
    }
    if constexpr (M == 2) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
                     "r"(r[2]), "r"(r[3])
                     : "memory");
    } else if constexpr (M == 4) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                     : "memory");
    } else {
        static_assert(M == 8, "tmem_st_vec: M in {2,4,8}");
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
            "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
            : "memory");
    }
}

template <int M>
__device__ __forceinline__ void tmem_ld_vec(uint32_t taddr, double (&v)[M]) {
    uint32_t r[2 * M];
    if constexpr (M == 2) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(taddr)
                     : "memory");
    } else if constexpr (M == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr)
                     : "memory");
    } else {
        static_assert(M == 8, "tmem_ld_vec: M in {2,4,8}");
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr)
            : "memory");
    }
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}

// Per-point epilogue of the apply phase.  Returns the value written to the output slab
// (marginal / new phi_k), accumulates residual / cost partial sums, flags loss of range.
template <int NB, typename T, int MODE>
__device__ __forceinline__ double epilogue(const T &J, const double *cur, int lane, int jx, double &acc, bool &bad) {
    using AV = ApplyVecs<NB, MODE>;
    constexpr int S = slab_s(NB);
    const double jv = value_of(J);
    if (MODE == MODE_MARG) {
        const double ph = cur[(AV::IPHI * 32 + lane) * (S + 1) + jx];
        bad |= ph > 0.0 && !finite_positive(jv);  // J left the fp64 range (all terms are positive)
        return ph * jv;
    } else if (MODE == MODE_UPD) {
        const double mu = cur[(AV::IMU * 32 + lane) * (S + 1) + jx];
        const double q = div_nr1(mu, jv);
        const bool nz = nonzero(mu);
        bad |= nz && !finite_positive(q);  // J = 0 / inf / NaN or mu/J out of range
        return nz ? q : 0.0;
    } else if (MODE == MODE_RES) {
        const double ph = cur[(AV::IPHI * 32 + lane) * (S + 1) + jx];
        bad |= ph > 0.0 && !finite_positive(jv);
        acc += fabs(ph * jv - cur[(AV::IMU * 32 + lane) * (S + 1) + jx]);
        return 0.0;
    } else {
        const double ph = cur[(AV::IPHI * 32 + lane) * (S + 1) + jx];
        bad |= ph > 0.0 && !finite_positive(jv);
        if constexpr (sizeof(T) == sizeof(Dual)) acc += ph * reinterpret_cast<const Dual &>(J).d;
        return 0.0;
    }
}

// NEXT-1 (MODE_ALLRES): with the states of the DP over ALL l scalings (NB = l), the states without
// marginal k are exactly update k's states, so every J_k at this point is the combine over the
// subsets S of A_k = {0..l-1} minus k:  J_k = sum_{S in A_k} F[S] H[A_k \ S]  (H = D B_{m+1}: the
// combine weight w_{|S|+1} = w_{l-1-|S|} is D's entry of A_k \ S).  Returns sum_{k<l-1} |phi_k J_k - mu_k|
// (Algorithm 1 line 7, generalised) from one pass instead of l-1 products.
template <int NB, int SL, typename T>
__device__ __forceinline__ double allres_terms(const T (&F)[1 << NB], const T (&H)[1 << NB],
                                               const double (&f)[NB > 0 ? NB : 1], const double *cur, int lane, int jx,
                                               bool &bad) {
    constexpr int M = 1 << NB;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k + 1 < NB; ++k) {
        double J = 0.0;
#pragma unroll
        for (int S = 0; S < M; ++S)
            if (!((S >> k) & 1)) J = fma(value_of(F[S]), value_of(H[(M - 1) & ~S & ~(1 << k)]), J);
        const double ph = f[k];
        bad |= ph > 0.0 && !finite_positive(J);
        s += fabs(ph * J - cur[((NB + k) * 32 + lane) * (SL + 1) + jx]);
    }
    return s;
}

// Next-update operator step (fused): the bound values of update k+1 at this point, cyclic bound
// order (see make_plan); one extended operator walk gives both scan directions (dp.cuh opx_*).
template <int NB, typename T>
__device__ __forceinline__ void next_ops_step(T (&Gx)[NB + 1][1 << NB], const T *wt, const double (&f)[NB > 0 ? NB : 1],
                                              double phi, bool first) {
    double fn[NB > 0 ? NB : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b) fn[b] = b + 1 < NB ? f[b + 1] : phi;
    opx_step<NB, T>(Gx, wt, fn, first);
}

// FULL = every live lane owns a complete chain of P points (P % S == 0): no per-point bounds
// predicates, compile-time checkpoint positions.  The ragged last chain (and tiny P) use
// FULL = false.  Chains [cbeg, cend) are processed.
template <int NB, typename T, int MODE, bool NEXT, bool FULL, bool PTS = false>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_chunk_apply(Plan p, int64_t cbeg, int64_t cend) {
    using AV = ApplyVecs<NB, MODE>;
    constexpr int M = 1 << NB;
    constexpr int Q = sub_q(NB);
    constexpr int NSUB = nsub_max(NB);
    constexpr int S = slab_s(NB);
    constexpr int QPS = S / Q;
    constexpr int TILE = 32 * (S + 1);
    constexpr int NV = AV::NV;
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t chain0 = cbeg + ((int64_t)blockIdx.x * kWarpsPerCta + warp) * 32;
    if (chain0 >= cend || *p.stop) return;
    double *buf = smem + (size_t)warp * (2 * NV + 1) * TILE;
    double *obuf = buf + 2 * NV * TILE;
    const int64_t c = chain0 + lane;
    const bool live = c < cend;
    const int64_t x0 = c * p.P;
    const int64_t x1 = FULL ? x0 + p.P : min(p.N, x0 + p.P);
    const int ns = (int)((p.P + S - 1) / S);
    const double *vecs[NV];
#pragma unroll
    for (int b = 0; b < NB; ++b) vecs[b] = p.bound[b];
    if (AV::kMu) vecs[AV::IMU] = p.muk;
    if (AV::kPhi) vecs[AV::IPHI] = p.phik;
    if constexpr (MODE == MODE_ALLRES) {
#pragma unroll
        for (int k = 0; k + 1 < NB; ++k) vecs[NB + k] = p.mus[k];
    }
    T wt[NB + 2];
    load_weights<NB, T>(wt, p.W);
    T F[M], st[M];
    if (live) {
        vec_load<NB, T>(F, static_cast<const T *>(p.car_f[0]) + c * M);
        vec_load<NB, T>(st, static_cast<const T *>(p.car_b[0]) + c * M);
    } else {
        vec_unit<NB, T>(F);
        vec_unit<NB, T>(st);
    }
    double f[NB > 0 ? NB : 1];
    T Gx[NEXT ? NB + 1 : 1][NEXT ? M : 1];
    if constexpr (NEXT) opx_identity<NB, T>(Gx);
    // ---- walk 1 (right to left): suffix states, checkpoint ck[j] = B at min(x0+(j+1)Q, x1) ----
    T ck[NSUB][M];
    if (FULL) {
#pragma unroll
        for (int S2 = 0; S2 < M; ++S2) ck[p.P / Q - 1][S2] = st[S2];
    } else if (live && x1 > x0) {
        const int jl = (int)((x1 - 1 - x0) / Q);
#pragma unroll
        for (int S2 = 0; S2 < M; ++S2) ck[jl][S2] = st[S2];
    }
    slab_issue<S, NB>(buf, vecs, chain0, p.P, p.N, ns - 1, lane);
    cp_async_commit();
#pragma unroll 1
    for (int t = 0; t < ns; ++t) {
        const int s = ns - 1 - t;
        if (s > 0) slab_issue<S, NB>(buf + ((t + 1) & 1) * NV * TILE, vecs, chain0, p.P, p.N, s - 1, lane);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const double *cur = buf + (t & 1) * NV * TILE;
#pragma unroll
        for (int jj = S - 1; jj >= 0; --jj) {
            if (FULL) {
                if (jj == 0 && s == 0) break;
                slab_f<NB, S>(f, cur, lane, jj);
                diag_e<NB, T, PTS>(st, wt, p, x0 + (int64_t)s * S + jj + 1);
                dp_place<NB, T>(st, f);
                if (jj % Q == 0) {
                    const int j = s * QPS + jj / Q - 1;
#pragma unroll
                    for (int S2 = 0; S2 < M; ++S2) ck[j][S2] = st[S2];
                }
            } else {
                const int64_t x = x0 + (int64_t)s * S + jj;
                if (x < x1 && x > x0) {
                    slab_f<NB, S>(f, cur, lane, jj);
                    diag_e<NB, T, PTS>(st, wt, p, x + 1);
                    dp_place<NB, T>(st, f);
                    if ((((int)(x - x0)) % Q) == 0) {
                        const int j = (int)((x - x0) / Q) - 1;
#pragma unroll
                        for (int S2 = 0; S2 < M; ++S2) ck[j][S2] = st[S2];
                    }
                }
            }
        }
        __syncwarp();
    }
    // ---- walk 2 (left to right): rebuild suffix states per Q-block, prefix step, combine ----
    double acc = 0.0;
    bool bad = false;
    slab_issue<S, NV>(buf, vecs, chain0, p.P, p.N, 0, lane);
    cp_async_commit();
#pragma unroll 1
    for (int s = 0; s < ns; ++s) {
        if (s + 1 < ns) slab_issue<S, NV>(buf + ((s + 1) & 1) * NV * TILE, vecs, chain0, p.P, p.N, s + 1, lane);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const double *cur = buf + (s & 1) * NV * TILE;
#pragma unroll
        for (int jb = 0; jb < QPS; ++jb) {
            const int64_t base = x0 + (int64_t)s * S + jb * Q;
            const int len = FULL ? Q : (int)max((int64_t)0, min((int64_t)Q, x1 - base));
            if (FULL || len > 0) {
                T H[Q][M];
#pragma unroll
                for (int S2 = 0; S2 < M; ++S2) st[S2] = ck[s * QPS + jb][S2];
#pragma unroll
                for (int i = Q - 1; i >= 0; --i) {
                    if (FULL || i < len) {
                        diag_e<NB, T, PTS>(st, wt, p, base + i + 1);
#pragma unroll
                        for (int S2 = 0; S2 < M; ++S2) H[i][S2] = st[S2];
                        if (i > 0) {
                            slab_f<NB, S>(f, cur, lane, jb * Q + i);
                            dp_place<NB, T>(st, f);
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    if (FULL || i < len) {
                        const int jx = jb * Q + i;
                        slab_f<NB, S>(f, cur, lane, jx);
                        diag_e<NB, T, PTS>(F, wt, p, base + i);
                        dp_place<NB, T>(F, f);
                        if constexpr (MODE == MODE_ALLRES) {
                            acc += allres_terms<NB, S>(F, H[i], f, cur, lane, jx, bad);
                        } else {
                            const T J = combine<NB, T>(F, H[i]);
                            const double o = epilogue<NB, T, MODE>(J, cur, lane, jx, acc, bad);
                            if (AV::kOut) obuf[lane * (S + 1) + jx] = o;
                            if constexpr (NEXT) next_ops_step<NB, T>(Gx, wt, f, o, s == 0 && jb == 0 && i == 0);
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (AV::kOut) {
            slab_store<S>(obuf, p.outk, chain0, cend, p.P, p.N, s, lane);
            __syncwarp();
        }
    }
    if (bad && live) raise_status(p, 6 /*EOVERFLOW*/);
    if ((MODE == MODE_RES || MODE == MODE_COST || MODE == MODE_ALLRES) && live) p.partial[c] = acc;
    if constexpr (NEXT) {
        if (live) {
            opx_store<NB, T>(Gx, wt, static_cast<T *>(p.ops_f[0]) + c * OpShape<NB>::SZ,
                             static_cast<T *>(p.ops_b[0]) + c * OpShape<NB>::SZ);
        }
    }
}

// FULL-chain apply with the suffix checkpoints in TMEM (fp64, NB <= 3).  Walk 1 (right to left)
// stores B at every 2Q-block end (one slab = one 2Q-block).  Walk 2 (left to right), per block:
// reload B_end from TMEM, walk the right half back to get B_mid (Q extra steps), rebuild the
// left half's suffix states from B_mid and run the prefix/combine/epilogue over it, then the
// same for the right half from B_end.
template <int NB, int MODE, bool NEXT>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_chunk_apply_tm(Plan p, int64_t cbeg, int64_t cend) {
    using T = double;
    using AV = ApplyVecs<NB, MODE>;
    constexpr int M = 1 << NB;
    constexpr int Q = sub_q(NB);
    constexpr int Q2 = 2 * Q;
    constexpr int S = slab_s(NB);
    static_assert(S == Q2, "one slab per checkpoint block");
    constexpr int TILE = 32 * (S + 1);
    constexpr int NV = AV::NV;
    __shared__ uint32_t tmem_slot;
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t chain0 = cbeg + ((int64_t)blockIdx.x * kWarpsPerCta + warp) * 32;
    const bool active = chain0 < cend && !*(volatile int *)p.stop;
    if (warp == 0) tmem_alloc(&tmem_slot);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = tmem_slot + ((uint32_t)(32 * warp) << 16);
    if (active) {
        double *buf = smem + (size_t)warp * (2 * NV + 1) * TILE;
        double *obuf = buf + 2 * NV * TILE;
        const int64_t c = chain0 + lane;
        const bool live = c < cend;
        const int ns = (int)(p.P / S);
        const double *vecs[NV];
#pragma unroll
        for (int b = 0; b < NB; ++b) vecs[b] = p.bound[b];
        if (AV::kMu) vecs[AV::IMU] = p.muk;
        if (AV::kPhi) vecs[AV::IPHI] = p.phik;
        T wt[NB + 2];
        load_weights<NB, T>(wt, p.W);
        T F[M], st[M];
        if (live) {
            vec_load<NB, T>(F, static_cast<const T *>(p.car_f[0]) + c * M);
            vec_load<NB, T>(st, static_cast<const T *>(p.car_b[0]) + c * M);
        } else {
            vec_unit<NB, T>(F);
            vec_unit<NB, T>(st);
        }
        double f[NB > 0 ? NB : 1];
        T Gx[NEXT ? NB + 1 : 1][NEXT ? M : 1];
        if constexpr (NEXT) opx_identity<NB, T>(Gx);
        // ---- walk 1: right to left, checkpoint B at every block end into TMEM ----
        slab_issue<S, NB>(buf, vecs, chain0, p.P, p.N, ns - 1, lane);
        cp_async_commit();
#pragma unroll 1
        for (int t = 0; t < ns; ++t) {
            const int s = ns - 1 - t;
            tmem_st_vec<M>(tbase + (uint32_t)(s * 2 * M), st);
            if (s > 0) slab_issue<S, NB>(buf + ((t + 1) & 1) * NV * TILE, vecs, chain0, p.P, p.N, s - 1, lane);
            cp_async_commit();
            if (s == 0) break;  // the state left of the chain is not needed
            cp_async_wait<1>();
            __syncwarp();
            const double *cur = buf + (t & 1) * NV * TILE;
#pragma unroll
            for (int jj = S - 1; jj >= 0; --jj) {
                slab_f<NB, S>(f, cur, lane, jj);
                dp_diag<NB, T, true>(st, wt);
                dp_place<NB, T>(st, f);
            }
            __syncwarp();
        }
        cp_async_wait<0>();
        __syncwarp();
        tmem_wait_st();
        // ---- walk 2: left to right ----
        double acc = 0.0;
        bool bad = false;
        slab_issue<S, NV>(buf, vecs, chain0, p.P, p.N, 0, lane);
        cp_async_commit();
#pragma unroll 1
        for (int s = 0; s < ns; ++s) {
            if (s + 1 < ns) slab_issue<S, NV>(buf + ((s + 1) & 1) * NV * TILE, vecs, chain0, p.P, p.N, s + 1, lane);
            cp_async_commit();
            T bend[M];
            tmem_ld_vec<M>(tbase + (uint32_t)(s * 2 * M), bend);
            cp_async_wait<1>();
            __syncwarp();
            const double *cur = buf + (s & 1) * NV * TILE;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                // suffix state at the right end of this half-block
#pragma unroll
                for (int S2 = 0; S2 < M; ++S2) st[S2] = bend[S2];
                if (half == 0) {
#pragma unroll
                    for (int i = Q2 - 1; i >= Q; --i) {
                        slab_f<NB, S>(f, cur, lane, i);
                        dp_diag<NB, T, true>(st, wt);
                        dp_place<NB, T>(st, f);
                    }
                }
                T H[Q][M];
#pragma unroll
                for (int i = Q - 1; i >= 0; --i) {
                    dp_diag<NB, T, true>(st, wt);
#pragma unroll
                    for (int S2 = 0; S2 < M; ++S2) H[i][S2] = st[S2];
                    if (i > 0) {
                        slab_f<NB, S>(f, cur, lane, half * Q + i);
                        dp_place<NB, T>(st, f);
                    }
                }
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    const int jx = half * Q + i;
                    slab_f<NB, S>(f, cur, lane, jx);
                    dp_diag<NB, T, true>(F, wt);
                    dp_place<NB, T>(F, f);
                    const T J = combine<NB, T>(F, H[i]);
                    const double o = epilogue<NB, T, MODE>(J, cur, lane, jx, acc, bad);
                    if (AV::kOut) obuf[lane * (S + 1) + jx] = o;
                    if constexpr (NEXT) next_ops_step<NB, T>(Gx, wt, f, o, s == 0 && half == 0 && i == 0);
                }
            }
            __syncwarp();
            if (AV::kOut) {
                slab_store<S>(obuf, p.outk, chain0, cend, p.P, p.N, s, lane);
                __syncwarp();
            }
        }
        if (bad && live) raise_status(p, 6 /*EOVERFLOW*/);
        if ((MODE == MODE_RES || MODE == MODE_COST) && live) p.partial[c] = acc;
        if constexpr (NEXT) {
            if (live) {
                opx_store<NB, T>(Gx, wt, static_cast<T *>(p.ops_f[0]) + c * OpShape<NB>::SZ,
                                 static_cast<T *>(p.ops_b[0]) + c * OpShape<NB>::SZ);
            }
        }
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(tmem_slot);
}

// ---------------------------------------------------------------------------------------
// Single-walk apply (stable regime: P * max_a a(l-a) * h/eta <= kSwBound, see mmot_create).
// Every chain is walked ONCE, left to right; each grid point is read from HBM once.
//   prefix:  F_m = place_m(D F_{m-1})                         (exact carry F_{x0-1} from the scan)
//   suffix:  U_m = place_m^{-1}(B_m) = D B_{m+1},  B_{m+1} = D^{-1} U_m
//            (exact inclusive carry B_{x0} from the scan; the inverse step is well conditioned
//             because D^{-1} = diag(w^{-1}) grows by at most e^{kSwBound} over a chain)
//   combine: J[m] = sum_S F_m[S] w_{|S|+1} B_{m+1}[S^c] = sum_S F_m[S] U_m[S^c]   (w_a = w_{l-a})
// The next update's chain operators come from ONE extended walk (opx_step, prefix/suffix
// duality in dp.cuh).
// ---------------------------------------------------------------------------------------
template <int NB, typename T>
__device__ __forceinline__ void load_winv(T (&wi)[NB + 2], const Weights &W) {
#pragma unroll
    for (int a = 0; a <= NB + 1; ++a) {
        double v;
        load_weight(v, W, a);
        const double r = 1.0 / v;
        if constexpr (sizeof(T) == sizeof(double)) {
            reinterpret_cast<double &>(wi[a]) = r;
        } else {
            // d(1/w)/dlog(lambda) = -e_a / w_a
            reinterpret_cast<Dual &>(wi[a]) = Dual{r, -W.e[a] * r};
        }
    }
}

// ---------------------------------------------------------------------------------------
// Chain-blocked transposed layout (single-walk contexts).  Chains are grouped by 32 (one warp);
// element (chain c, offset t) lives at (c/32)*32P + t*32 + c%32.  A warp's slab (S offsets of one
// vector for its 32 chains) is then S*256 contiguous bytes: ONE bulk copy (cp.async.bulk +
// mbarrier transaction count) per vector per slab, landing in shared memory as [NV][S][32]
// (conflict-free reads: lane r reads column r); outputs are stored straight from registers,
// 256 contiguous bytes per warp store.  Points beyond N (tail of the last chain, and the padding
// chains up to a multiple of 32) are zeros: phi = mu = 0 there contributes nothing to any carry
// that is used.
// ---------------------------------------------------------------------------------------
constexpr int kSwS = 8;      // offsets per slab
#ifndef MMOT_SW_STAGES
#define MMOT_SW_STAGES 3
#endif
#ifndef MMOT_SW_MINB3
#define MMOT_SW_MINB3 2
#endif
#ifndef MMOT_SW_SCL
#define MMOT_SW_SCL 1
#endif
constexpr int kSwStages = MMOT_SW_STAGES; // slab stages per warp (two in flight while one is consumed)

// Issue slab s (offsets s*S .. s*S+S-1) of NV vectors for the warp's 32 chains (block base
// offset wbase = chain0 * P) into stage buffer sbuf [NV][S][32]: NV bulk copies of S*256 bytes.
template <int NV>
__device__ __forceinline__ void sw_issue(double *sbuf, uint64_t *bar, const double *const *vecs, int64_t wbase, int s,
                                         int lane) {
    constexpr int S = kSwS;
    if (lane == 0) {
        mbar_arrive_expect_tx(bar, (uint32_t)(NV * S * 32 * sizeof(double)));
#pragma unroll
        for (int v = 0; v < NV; ++v)
            bulk_g2s(sbuf + v * S * 32, vecs[v] + wbase + (int64_t)s * S * 32, S * 32 * sizeof(double), bar);
    }
}

template <int NB>
__device__ __forceinline__ void rx_load(double (&E)[Rx<NB>::SZE], const double *src, int64_t i, int64_t n) {
    if (i < n) {
#pragma unroll
        for (int q = 0; q < Rx<NB>::SZE; ++q) E[q] = src[i * Rx<NB>::SZE + q];
    } else {
        rx_identity<NB>(E);
    }
}
template <int NB>
__device__ __forceinline__ void rx_shfl(double (&D)[Rx<NB>::SZE], const double (&E)[Rx<NB>::SZE], int delta, int mode) {
#pragma unroll
    for (int q = 0; q < Rx<NB>::SZE; ++q)
        D[q] = mode == 1 ? __shfl_up_sync(0xffffffffu, E[q], delta) : __shfl_down_sync(0xffffffffu, E[q], delta);
}

template <int NB, typename T, int MODE, bool NEXT, bool NXR = false>
__global__ void __launch_bounds__(kWarpsPerCta * 32, NB >= 4 ? 1 : (NB == 3 ? MMOT_SW_MINB3 : 2)) k_sw_apply(Plan p) {
    using AV = ApplyVecs<NB, MODE>;
    constexpr int M = 1 << NB;
    constexpr int S = kSwS;
    constexpr int NV = AV::NV;
    constexpr int STG = NV * S * 32;  // doubles per stage
    extern __shared__ __align__(128) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t chain0 = ((int64_t)blockIdx.x * kWarpsPerCta + warp) * 32;
    if (chain0 >= p.nchunks || *(volatile int *)p.stop) return;
    double *buf = smem + (size_t)warp * kSwStages * STG;
    __shared__ uint64_t bars[kWarpsPerCta][kSwStages];
    uint64_t *bar = bars[warp];
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kSwStages; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const int64_t c = chain0 + lane;
    const bool live = c < p.nchunks;
    const int ns = (int)(p.P / S);
    const double *vecs[NV];
#pragma unroll
    for (int b = 0; b < NB; ++b) vecs[b] = p.bound[b];
    if (AV::kMu) vecs[AV::IMU] = p.muk;
    if (AV::kPhi) vecs[AV::IPHI] = p.phik;
    T wt[NB + 2], wi[NB + 2];
    load_weights<NB, T>(wt, p.W);
    load_winv<NB, T>(wi, p.W);
    T F[M], B[M];
    if (live) {
        vec_load<NB, T>(F, static_cast<const T *>(p.car_f[0]) + c * M);
        vec_load<NB, T>(B, static_cast<const T *>(p.car_bi) + c * M);
    } else {
        vec_unit<NB, T>(F);
        vec_unit<NB, T>(B);
    }
    if constexpr (NXR) {
        // level 0 of the restricted scan, fused: the new-part carries of this warp's 32 chains from
        // the elements the previous update left in rxe_*[0] and the group carries of level 1
        if (p.rx_scan) {
            constexpr int SZE = Rx<NB>::SZE;
            constexpr int MOn = Rx<NB>::MO;
            constexpr int NEW = 1 << (NB - 1);
            const int64_t g = chain0 / 32;
#pragma unroll
            for (int dir = 0; dir < 2; ++dir) {
                double A[SZE], Bv[SZE], C[SZE];
                rx_load<NB>(A, static_cast<const double *>(dir == 0 ? p.rxe_f[0] : p.rxe_b[0]), c, p.nchunks);
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    rx_shfl<NB>(Bv, A, d, dir == 0 ? 1 : 2);
                    rx_compose<NB>(Bv, A, C);
                    const bool take = dir == 0 ? lane >= d : lane + d < 32;
                    if (take) {
#pragma unroll
                        for (int q = 0; q < SZE; ++q) A[q] = C[q];
                    }
                }
                double cin[MOn], out[MOn];
                const double *gc = p.nlev > 1 ? static_cast<const double *>(dir == 0 ? p.rcar_f[1] : p.rcar_b[1]) : nullptr;
#pragma unroll
                for (int U = 0; U < MOn; ++U) cin[U] = gc ? gc[g * MOn + U] : 0.0;
                rx_apply<NB>(A, cin, out);
#pragma unroll
                for (int U = 0; U < MOn; ++U) {
                    if (dir == 0) {
                        const double up = __shfl_up_sync(0xffffffffu, out[U], 1);
                        reinterpret_cast<double &>(F[U | NEW]) = lane == 0 ? cin[U] : up;  // exclusive prefix
                    } else {
                        reinterpret_cast<double &>(B[U | NEW]) = out[U];                   // inclusive suffix
                        // complete this chain's carry in car_bi (read by the precision guard)
                        if (live && p.guard) static_cast<double *>(p.car_bi)[c * M + (U | NEW)] = out[U];
                    }
                }
            }
        }
    }
    T Gx[NEXT ? NB + 1 : 1][NEXT ? M : 1];
    if constexpr (NEXT) opx_identity<NB, T>(Gx);
    // restricted next-update scan elements (dp.cuh Rx): L, running Gr, M; old parts of the carries
    constexpr int MO = NXR ? Rx<NB>::MO : 1;
    double rL[MO], rM[MO], rG[NXR ? NB : 1][MO];
    // rG is kept scaled by rgs = w_1^t (rx_G_step_scaled); rwr[a] = w_a / w_1
    double rgs = 1.0, rwr[NB + 2];
#pragma unroll
    for (int a = 0; a <= NB + 1; ++a) rwr[a] = value_of(wt[a]) / value_of(wt[1]);
    const double rw1inv = 1.0 / value_of(wt[1]);
    if constexpr (NXR) {
#pragma unroll
        for (int U = 0; U < MO; ++U) {
            rL[U] = 0.0;
            rM[U] = 0.0;
#pragma unroll
            for (int c = 0; c < NB; ++c) rG[c][U] = U == 0 ? 1.0 : 0.0;
        }
        if (live) {
            double *nf = static_cast<double *>(p.ncar_f) + c * M;
            double *nb = static_cast<double *>(p.ncar_bi) + c * M;
#pragma unroll
            for (int U = 0; U < MO; ++U) {
                nf[U] = value_of(F[U << 1]);
                nb[U] = value_of(B[U << 1]);
            }
        }
    }
    // Scaled frames (fp64): the prefix states are kept as F~ = F w_1^{-t} and the suffix states as
    // B~ = B w_1^{t} (t = points walked, counting the diag of the edge entering the chain), so the
    // per-level diag multipliers become w_a / w_1 and w_1 / w_a -- exactly 1 for |S| in {1, l-1}
    // (w_{l-1} = w_1): those states need no multiply -- while the combine sum_S F~[S] U~[S^c] is J
    // itself (the scales cancel).  DESIGN.md §5.
    constexpr bool SCL = MMOT_SW_SCL && sizeof(T) == sizeof(double);
    double cF[NB + 2], cB[NB + 2];
    if constexpr (SCL) {
        const double w1 = value_of(wt[1]);
#pragma unroll
        for (int a = 0; a <= NB + 1; ++a) {
            cF[a] = a == 0 ? rw1inv : rwr[a];
            cB[a] = a == 0 ? w1 : 1.0 / rwr[a];
        }
#pragma unroll
        for (int S = 0; S < M; ++S) reinterpret_cast<double &>(B[S]) *= w1;
    }
    // the next-update operator step of point m is issued after the scans of point m+1
    // (software pipelining: the division of point m overlaps the scans of point m+1)
    double fprev[NB > 0 ? NB : 1], oprev = 0.0;
    bool have_prev = false;
    double acc = 0.0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < kSwStages - 1; ++i)
        if (i < ns) sw_issue<NV>(buf + i * STG, &bar[i], vecs, chain0 * p.P, i, lane);
#pragma unroll 1
    for (int s = 0; s < ns; ++s) {
        {
            const int sn = s + kSwStages - 1;  // refill the stage consumed in iteration s-1
            if (sn < ns) sw_issue<NV>(buf + (sn % kSwStages) * STG, &bar[sn % kSwStages], vecs, chain0 * p.P, sn, lane);
        }
        mbar_wait(&bar[s % kSwStages], (uint32_t)((s / kSwStages) & 1));
        const double *cur = buf + (s % kSwStages) * STG;
        double *outp = AV::kOut ? p.outk + chain0 * p.P + (int64_t)s * S * 32 + lane : nullptr;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            double f[NB > 0 ? NB : 1];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = cur[(b * S + j) * 32 + lane];
            if constexpr (SCL) dp_diag_lvl<NB>(reinterpret_cast<double(&)[M]>(F), cF);
            else dp_diag<NB, T, true>(F, wt);
            dp_place<NB, T>(F, f);
            double Bo[MO];
            if constexpr (NXR) {
#pragma unroll
                for (int U = 0; U < MO; ++U) Bo[U] = value_of(B[U << 1]);
            }
            dp_unplace<NB, T>(B, f);          // B := U_m = D B_{m+1}
            const T J = combine<NB, T>(F, B);
            if constexpr (SCL) dp_diag_lvl<NB>(reinterpret_cast<double(&)[M]>(B), cB);
            else dp_diag_inv<NB, T>(B, wi);   // B := B_{m+1}
            if constexpr (NEXT) {
                if (j > 0 || have_prev) next_ops_step<NB, T>(Gx, wt, fprev, oprev, j == 1 && s == 0);
            }
            const double jv = value_of(J);
            double o = 0.0;
            if (MODE == MODE_MARG) {
                const double ph = cur[(AV::IPHI * S + j) * 32 + lane];
                bad |= ph > 0.0 && !finite_positive(jv);  // J left the fp64 range
                o = ph * jv;
            } else if (MODE == MODE_UPD) {
                const double mu = cur[(AV::IMU * S + j) * 32 + lane];
                const double q = div_nr0(mu, jv);  // 2^-46 relative: inside the 1e-10 parity tolerance
                const bool nz = nonzero(mu);
                bad |= nz && !finite_positive(q);
                o = nz ? q : 0.0;
            } else if (MODE == MODE_RES) {
                const double ph = cur[(AV::IPHI * S + j) * 32 + lane];
                bad |= ph > 0.0 && !finite_positive(jv);
                acc += fabs(ph * jv - cur[(AV::IMU * S + j) * 32 + lane]);
            } else {
                const double ph = cur[(AV::IPHI * S + j) * 32 + lane];
                bad |= ph > 0.0 && !finite_positive(jv);
                if constexpr (sizeof(T) == sizeof(Dual)) acc += ph * reinterpret_cast<const Dual &>(J).d;
            }
            if (AV::kOut) outp[j * 32] = o;
            if constexpr (NEXT) {
#pragma unroll
                for (int b = 0; b < NB; ++b) fprev[b] = f[b];
                oprev = o;
            }
            if constexpr (NXR) {
                if constexpr (sizeof(T) == sizeof(double)) {
                    const bool first = j == 0 && s == 0;
                    if constexpr (SCL) {
                        // Bo is B~ = B w_1^{t}: o * Bo = w_1^2 (o * rgs * B) -- rM kept as M w_1
                        rx_M_acc_scaled<NB>(rM, rG, rwr, 1.0, o, Bo, first);
                    } else {
                        rx_M_acc_scaled<NB>(rM, rG, rwr, rw1inv, o * rgs, Bo, first);  // rM kept as M / w_1
                    }
                    rx_G_step_scaled<NB>(rG, rwr, f, first);
                    if (!first) rgs *= reinterpret_cast<const double *>(wt)[1];
                    if constexpr (SCL)  // L kept as L w_1^{-t}, like F
                        rx_L_step_scl<NB>(rL, rwr, f, o, reinterpret_cast<const double(&)[M]>(F));
                    else
                        rx_L_step<NB>(rL, reinterpret_cast<const double *>(wt), f, o, reinterpret_cast<const double(&)[M]>(F));
                }
            }
        }
        have_prev = true;
        __syncwarp();  // every lane is done with this stage before it is refilled
    }
    if constexpr (NEXT) {
        if (have_prev) next_ops_step<NB, T>(Gx, wt, fprev, oprev, ns == 1 && kSwS == 1);
    }
    if (bad && live) {
        raise_status(p, 6 /*EOVERFLOW*/);
        if (p.guard) atomicOr(p.guard, 1);  // may be the single walk's lost precision: redo on two-walk
    }
    if ((MODE == MODE_RES || MODE == MODE_COST) && live) p.partial[c] = acc;
    if (live && p.sw_end) {
        // walked suffix state after the chain's last point and the prefix state at that point
        T *e = static_cast<T *>(p.sw_end) + c * 2 * M;
        if constexpr (SCL) {
            // t = P at the chain end: F = F~ w_1^P, B = B~ w_1^{-(P+1)}
            const double w1 = value_of(wt[1]);
            const double wp = pow(w1, (double)p.P), wpi = 1.0 / (wp * w1);
#pragma unroll
            for (int R = 0; R < M; ++R) {
                e[R] = reinterpret_cast<const double &>(B[R]) * wpi;
                e[M + R] = reinterpret_cast<const double &>(F[R]) * wp;
            }
        } else {
#pragma unroll
            for (int R = 0; R < M; ++R) {
                e[R] = B[R];
                e[M + R] = F[R];
            }
        }
    }
    if constexpr (NEXT) {
        if (live)
            opx_store<NB, T>(Gx, wt, static_cast<T *>(p.ops_f[0]) + c * OpShape<NB>::SZ,
                             static_cast<T *>(p.ops_b[0]) + c * OpShape<NB>::SZ);
    }
    if constexpr (NXR) {
        constexpr int SZE = Rx<NB>::SZE;
        double ef[SZE], eb[SZE];
#pragma unroll
        for (int c = 0; c < NB; ++c)
#pragma unroll
            for (int U = 0; U < MO; ++U) rG[c][U] *= rgs;  // unscale the running operator
        if constexpr (SCL) {
            const double wp = rgs * value_of(wt[1]);  // w_1^P
#pragma unroll
            for (int U = 0; U < MO; ++U) {
                rM[U] *= rw1inv;  // rM was kept as M w_1
                rL[U] *= wp;      // rL as L w_1^{-P}
            }
        } else {
#pragma unroll
            for (int U = 0; U < MO; ++U) rM[U] *= value_of(wt[1]);  // and the suffix offset
        }
        rx_store<NB>(rG, rL, rM, reinterpret_cast<const double *>(wt), ef, eb);
        if (!live) {
            rx_identity<NB>(ef);
            rx_identity<NB>(eb);
        } else {
#pragma unroll
            for (int q = 0; q < SZE; ++q) {
                static_cast<double *>(p.rxe_f[0])[c * SZE + q] = ef[q];
                static_cast<double *>(p.rxe_b[0])[c * SZE + q] = eb[q];
            }
        }
        // level 0 -> 1 of the restricted scan, fused: shuffle-tree composition of the warp's 32
        if (p.nlev > 1) {
            double Bv[SZE], C[SZE];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                rx_shfl<NB>(Bv, ef, d, 2);
                rx_compose<NB>(ef, Bv, C);
                if ((lane & (2 * d - 1)) == 0) {
#pragma unroll
                    for (int q = 0; q < SZE; ++q) ef[q] = C[q];
                }
                rx_shfl<NB>(Bv, eb, d, 2);
                rx_compose<NB>(Bv, eb, C);
                if ((lane & (2 * d - 1)) == 0) {
#pragma unroll
                    for (int q = 0; q < SZE; ++q) eb[q] = C[q];
                }
            }
            if (lane == 0) {
                const int64_t g = chain0 / 32;
#pragma unroll
                for (int q = 0; q < SZE; ++q) {
                    static_cast<double *>(p.rxe_f[1])[g * SZE + q] = ef[q];
                    static_cast<double *>(p.rxe_b[1])[g * SZE + q] = eb[q];
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// Affine scan of the restricted next-update elements (one warp per group of 32, shuffles).
// ---------------------------------------------------------------------------------------
template <int NB>
__global__ void __launch_bounds__(128) k_rx_reduce_w(const double *in_f, const double *in_b, double *out_f, double *out_b,
                                                    int64_t n_in, const int *stop) {
    constexpr int SZE = Rx<NB>::SZE;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t g = (int64_t)blockIdx.x * 4 + warp;
    const int dir = blockIdx.y;
    const int64_t first = g * 32;
    if (first >= n_in || *stop) return;
    double A[SZE], Bv[SZE], C[SZE];
    rx_load<NB>(A, dir == 0 ? in_f : in_b, first + lane, n_in);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        rx_shfl<NB>(Bv, A, d, 2);
        if (dir == 0) rx_compose<NB>(A, Bv, C);   // prefix: lower chain first
        else rx_compose<NB>(Bv, A, C);            // suffix: higher chain first
        if ((lane & (2 * d - 1)) == 0) {
#pragma unroll
            for (int q = 0; q < SZE; ++q) A[q] = C[q];
        }
    }
    if (lane == 0) {
        double *o = (dir == 0 ? out_f : out_b) + g * SZE;
#pragma unroll
        for (int q = 0; q < SZE; ++q) o[q] = A[q];
    }
}

// Down-sweep: group carries gc (MO per group, nullptr = zero new part at the top), member carries
// out: level >= 1 -> car (MO per member, exclusive in both directions); level 0 -> the full carry
// arrays (stride M, new-part positions U | newbit): prefix exclusive, suffix inclusive.
template <int NB>
__global__ void __launch_bounds__(128) k_rx_down_w(const double *el_f, const double *el_b, const double *gc_f,
                                                  const double *gc_b, double *car_f, double *car_b, int64_t n_in,
                                                  const int *stop, double *full_f, double *full_bi) {
    constexpr int SZE = Rx<NB>::SZE;
    constexpr int MO = Rx<NB>::MO;
    constexpr int M = 1 << NB;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t g = (int64_t)blockIdx.x * 4 + warp;
    const int dir = blockIdx.y;
    const int64_t first = g * 32;
    if (first >= n_in || *stop) return;
    double A[SZE], Bv[SZE], C[SZE];
    rx_load<NB>(A, dir == 0 ? el_f : el_b, first + lane, n_in);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        rx_shfl<NB>(Bv, A, d, dir == 0 ? 1 : 2);
        rx_compose<NB>(Bv, A, C);  // the earlier-applied part (from the shuffle) first
        const bool take = dir == 0 ? lane >= d : lane + d < 32;
        if (take) {
#pragma unroll
            for (int q = 0; q < SZE; ++q) A[q] = C[q];
        }
    }
    const double *gc = dir == 0 ? gc_f : gc_b;
    double cin[MO], out[MO], nb[MO];
#pragma unroll
    for (int U = 0; U < MO; ++U) cin[U] = gc ? gc[g * MO + U] : 0.0;
    rx_apply<NB>(A, cin, out);
#pragma unroll
    for (int U = 0; U < MO; ++U)
        nb[U] = dir == 0 ? __shfl_up_sync(0xffffffffu, out[U], 1) : __shfl_down_sync(0xffffffffu, out[U], 1);
    const bool edge = dir == 0 ? lane == 0 : lane == 31;
    const int64_t i = first + lane;
    if (i < n_in) {
        if (full_f) {  // level 0
            constexpr int NEW = 1 << (NB - 1);
            if (dir == 0) {
#pragma unroll
                for (int U = 0; U < MO; ++U) full_f[i * M + (U | NEW)] = edge ? cin[U] : nb[U];
            } else {
#pragma unroll
                for (int U = 0; U < MO; ++U) full_bi[i * M + (U | NEW)] = out[U];
            }
        } else {
            double *dst = (dir == 0 ? car_f : car_b) + i * MO;
#pragma unroll
            for (int U = 0; U < MO; ++U) dst[U] = edge ? cin[U] : nb[U];
        }
    }
}

// The top of the restricted scan in ONE launch (single-process contexts with >= 3 levels): the
// reduce of level top-1 (<= 1024 elements) into the <= 32 top elements, the down-sweep of the top
// level (zero new part entering it) and the down-sweep of level top-1, the top level's elements and
// carries staying in shared memory.  One CTA per direction; replaces three dependent launches of
// ~5 us each per update (C4: 74 -> 3 elements).  Same arithmetic, same order as k_rx_reduce_w /
// k_rx_down_w (bit-identical carries).
template <int NB>
__global__ void __launch_bounds__(128) k_rx_top(const double *e1_f, const double *e1_b, double *car1_f, double *car1_b,
                                               int64_t n1, const int *stop) {
    constexpr int SZE = Rx<NB>::SZE;
    constexpr int MO = Rx<NB>::MO;
    __shared__ double s_el[32][SZE];
    __shared__ double s_car[32][MO];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int dir = blockIdx.x;
    if (*stop) return;
    const int ng = (int)((n1 + 31) / 32);  // groups of level top-1 = elements of the top level (<= 32)
    const double *e1 = dir == 0 ? e1_f : e1_b;
    double A[SZE], Bv[SZE], C[SZE];
    for (int g = warp; g < ng; g += 4) {  // reduce: one top element per group
        rx_load<NB>(A, e1, (int64_t)g * 32 + lane, n1);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            rx_shfl<NB>(Bv, A, d, 2);
            if (dir == 0) rx_compose<NB>(A, Bv, C);
            else rx_compose<NB>(Bv, A, C);
            if ((lane & (2 * d - 1)) == 0) {
#pragma unroll
                for (int q = 0; q < SZE; ++q) A[q] = C[q];
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < SZE; ++q) s_el[g][q] = A[q];
        }
    }
    __syncthreads();
    if (warp == 0) {  // down-sweep of the top level: carries entering each group
        if (lane < ng) {
#pragma unroll
            for (int q = 0; q < SZE; ++q) A[q] = s_el[lane][q];
        } else {
            rx_identity<NB>(A);
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            rx_shfl<NB>(Bv, A, d, dir == 0 ? 1 : 2);
            rx_compose<NB>(Bv, A, C);
            const bool take = dir == 0 ? lane >= d : lane + d < 32;
            if (take) {
#pragma unroll
                for (int q = 0; q < SZE; ++q) A[q] = C[q];
            }
        }
        double cin[MO], out[MO], nb[MO];
#pragma unroll
        for (int U = 0; U < MO; ++U) cin[U] = 0.0;
        rx_apply<NB>(A, cin, out);
#pragma unroll
        for (int U = 0; U < MO; ++U)
            nb[U] = dir == 0 ? __shfl_up_sync(0xffffffffu, out[U], 1) : __shfl_down_sync(0xffffffffu, out[U], 1);
        const bool edge = dir == 0 ? lane == 0 : lane == 31;
        if (lane < ng) {
#pragma unroll
            for (int U = 0; U < MO; ++U) s_car[lane][U] = edge ? cin[U] : nb[U];
        }
    }
    __syncthreads();
    for (int g = warp; g < ng; g += 4) {  // down-sweep of level top-1
        const int64_t i = (int64_t)g * 32 + lane;
        rx_load<NB>(A, e1, i, n1);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            rx_shfl<NB>(Bv, A, d, dir == 0 ? 1 : 2);
            rx_compose<NB>(Bv, A, C);
            const bool take = dir == 0 ? lane >= d : lane + d < 32;
            if (take) {
#pragma unroll
                for (int q = 0; q < SZE; ++q) A[q] = C[q];
            }
        }
        double cin[MO], out[MO], nb[MO];
#pragma unroll
        for (int U = 0; U < MO; ++U) cin[U] = s_car[g][U];
        rx_apply<NB>(A, cin, out);
#pragma unroll
        for (int U = 0; U < MO; ++U)
            nb[U] = dir == 0 ? __shfl_up_sync(0xffffffffu, out[U], 1) : __shfl_down_sync(0xffffffffu, out[U], 1);
        const bool edge = dir == 0 ? lane == 0 : lane == 31;
        if (i < n1) {
            double *dst = (dir == 0 ? car1_f : car1_b) + i * MO;
#pragma unroll
            for (int U = 0; U < MO; ++U) dst[U] = edge ? cin[U] : nb[U];
        }
    }
}

// Levels >= 1 (level 0 is fused into the update kernels: reduce at the end of update k, down at
// the start of update k+1).
template <int NB>
__global__ void k_rx_compose(const double *all, int world, int rank, double *car) {
    if (threadIdx.x == 0) compose_rank_affine<NB>(all, world, rank, car, car + Rx<NB>::MO);
}

template <int NB>
static void launch_rx_scan(const Plan &p, cudaStream_t s, int64_t *launches) {
    static const bool no_top = getenv("MMOT_NO_RXTOP") != nullptr;
    const bool fuse_top = !p.exch && p.nlev >= 3 && !no_top;  // top two levels in one launch (k_rx_top)
    const int nred = fuse_top ? p.nlev - 2 : p.nlev - 1;
    for (int i = 1; i < nred; ++i) {
        const int64_t ng = p.nlev_n[i + 1];
        k_rx_reduce_w<NB><<<dim3((unsigned)((ng + 3) / 4), 2), 128, 0, s>>>(
            static_cast<const double *>(p.rxe_f[i]), static_cast<const double *>(p.rxe_b[i]),
            static_cast<double *>(p.rxe_f[i + 1]), static_cast<double *>(p.rxe_b[i + 1]), p.nlev_n[i], p.stop);
        ++*launches;
    }
    // sharded contexts: whole-shard affine elements (top level reduced to one), all-gathered,
    // composed into the new-part carries entering this shard
    const int top = p.nlev - 1;
    if (p.exch) {
        k_rx_reduce_w<NB><<<dim3(1, 2), 128, 0, s>>>(
            static_cast<const double *>(p.rxe_f[top]), static_cast<const double *>(p.rxe_b[top]),
            static_cast<double *>(p.agg_send), static_cast<double *>(p.agg_send) + Rx<NB>::SZE, p.nlev_n[top], p.stop);
        ++*launches;
        p.exch(p.exch_ctx, 2 * (size_t)Rx<NB>::SZE, s);
        k_rx_compose<NB><<<1, 1, 0, s>>>(static_cast<const double *>(p.agg_all), p.world, p.rank,
                                        static_cast<double *>(p.rank_car));
        ++*launches;
    }
    if (fuse_top) {
        const int t1 = p.nlev - 2;
        k_rx_top<NB><<<2, 128, 0, s>>>(static_cast<const double *>(p.rxe_f[t1]), static_cast<const double *>(p.rxe_b[t1]),
                                       static_cast<double *>(p.rcar_f[t1]), static_cast<double *>(p.rcar_b[t1]),
                                       p.nlev_n[t1], p.stop);
        ++*launches;
    }
    for (int i = fuse_top ? p.nlev - 3 : p.nlev - 1; i >= 1; --i) {
        const int64_t ng = (p.nlev_n[i] + 31) / 32;
        const double *gf = i + 1 < p.nlev ? static_cast<const double *>(p.rcar_f[i + 1])
                                          : (p.exch ? static_cast<const double *>(p.rank_car) : nullptr);
        const double *gb = i + 1 < p.nlev ? static_cast<const double *>(p.rcar_b[i + 1])
                                          : (p.exch ? static_cast<const double *>(p.rank_car) + Rx<NB>::MO : nullptr);
        k_rx_down_w<NB><<<dim3((unsigned)((ng + 3) / 4), 2), 128, 0, s>>>(
            static_cast<const double *>(p.rxe_f[i]), static_cast<const double *>(p.rxe_b[i]), gf, gb,
            static_cast<double *>(p.rcar_f[i]), static_cast<double *>(p.rcar_b[i]), p.nlev_n[i], p.stop,
            i == 0 ? static_cast<double *>(p.car_f[0]) : nullptr, i == 0 ? static_cast<double *>(p.car_bi) : nullptr);
        ++*launches;
    }
}

// Chain operators of a bound set in the transposed layout (first update of a solve).
template <int NB, typename T>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_sw_ops(Plan p) {
    constexpr int M = 1 << NB;
    constexpr int S = kSwS;
    constexpr int NV = NB;
    constexpr int STG = NV * S * 32;
    extern __shared__ __align__(128) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t chain0 = ((int64_t)blockIdx.x * kWarpsPerCta + warp) * 32;
    if (chain0 >= p.nchunks || *(volatile int *)p.stop) return;
    double *buf = smem + (size_t)warp * kSwStages * STG;
    __shared__ uint64_t bars[kWarpsPerCta][kSwStages];
    uint64_t *bar = bars[warp];
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kSwStages; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const int64_t c = chain0 + lane;
    const int ns = (int)(p.P / S);
    const double *vecs[NV];
#pragma unroll
    for (int b = 0; b < NB; ++b) vecs[b] = p.bound[b];
    T wt[NB + 2];
    load_weights<NB, T>(wt, p.W);
    T G[NB + 1][M];
    opx_identity<NB, T>(G);
#pragma unroll
    for (int i = 0; i < kSwStages - 1; ++i)
        if (i < ns) sw_issue<NV>(buf + i * STG, &bar[i], vecs, chain0 * p.P, i, lane);
#pragma unroll 1
    for (int s = 0; s < ns; ++s) {
        const int sn = s + kSwStages - 1;
        if (sn < ns) sw_issue<NV>(buf + (sn % kSwStages) * STG, &bar[sn % kSwStages], vecs, chain0 * p.P, sn, lane);
        mbar_wait(&bar[s % kSwStages], (uint32_t)((s / kSwStages) & 1));
        const double *cur = buf + (s % kSwStages) * STG;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            double f[NB > 0 ? NB : 1];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = cur[(b * S + j) * 32 + lane];
            opx_step<NB, T>(G, wt, f, s == 0 && j == 0);
        }
        __syncwarp();
    }
    if (c < p.nchunks)
        opx_store<NB, T>(G, wt, static_cast<T *>(p.ops_f[0]) + c * OpShape<NB>::SZ,
                         static_cast<T *>(p.ops_b[0]) + c * OpShape<NB>::SZ);
}

// Natural <-> chain-blocked layout: natural x = c*P + t  <->  (c/32)*32P + t*32 + c%32.
// op: 0 copy, 1 exp (natural log-scalings -> linear), 2 log (linear -> log-scalings).
// One CTA per 32 chains x 32 offsets tile (blockIdx.y = chain group).
// flags != nullptr: the input check of launch_check fused into the pass (bit0 NaN/Inf, bit1
// negative; -inf allowed when allow_neg_inf) and, if mass != nullptr, the sum of the inputs.
// Tile = 32 chains x 32 offsets, 128 threads: each thread loads its 8 elements before any use (8
// loads in flight per thread), then the tile is written transposed.  The natural-layout side reads
// 32 rows of 256 contiguous bytes, the chain-blocked side writes 8 KB contiguous.
constexpr int kTR = 4;  // thread rows per tile (blockDim.y)
__global__ void __launch_bounds__(32 * kTR) k_to_t(const double *__restrict__ src, double *__restrict__ dst, int64_t N,
                                                  int64_t P, int64_t nchains, int op, int *flags, double *mass,
                                                  int allow_neg_inf) {
    __shared__ double tile[32][33];
    __shared__ double msum[kTR];
    const int64_t t0 = (int64_t)blockIdx.x * 32, g = blockIdx.y, c0 = g * 32;
    constexpr int R = 32 / kTR;
    double v[R];
    const int64_t t = t0 + threadIdx.x;
#pragma unroll
    for (int i = 0; i < R; ++i) {  // r = chain within the tile, threadIdx.x = offset t
        const int64_t c = c0 + threadIdx.y + i * kTR;
        const int64_t x = c * P + t;
        v[i] = (c < nchains && t < P && x < N) ? __ldcs(src + x) : 0.0;
    }
    int fl = 0;
    double a = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int64_t c = c0 + threadIdx.y + i * kTR;
        const bool in = c < nchains && t < P && c * P + t < N;
        double x = v[i];
        if (flags && in) {
            if (isnan(x) || (isinf(x) && !(allow_neg_inf && x < 0))) fl |= 1;
            else if (x < 0 && !allow_neg_inf) fl |= 2;
            else if (!allow_neg_inf) a += x;
        }
        if (op == 1 && in) x = exp(x);
        tile[threadIdx.y + i * kTR][threadIdx.x] = x;
    }
    if (flags) {
        if (fl) atomicOr(flags, fl);
        if (mass) {
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) a += __shfl_xor_sync(0xffffffffu, a, d);
            if (threadIdx.x == 0) msum[threadIdx.y] = a;
        }
    }
    __syncthreads();
    if (flags && mass && threadIdx.y == 0 && threadIdx.x == 0) {
        double b = 0.0;
#pragma unroll
        for (int i = 0; i < kTR; ++i) b += msum[i];
        atomicAdd(mass, b);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {  // r = offset within the tile, threadIdx.x = chain
        const int64_t tt = t0 + threadIdx.y + i * kTR;
        if (tt < P) __stcs(dst + g * 32 * P + tt * 32 + threadIdx.x, tile[threadIdx.x][threadIdx.y + i * kTR]);
    }
}

__global__ void __launch_bounds__(32 * kTR) k_from_t(const double *__restrict__ src, double *__restrict__ dst,
                                                    int64_t N, int64_t P, int64_t nchains, int op) {
    __shared__ double tile[32][33];
    const int64_t t0 = (int64_t)blockIdx.x * 32, g = blockIdx.y, c0 = g * 32;
    constexpr int R = 32 / kTR;
    double v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {  // r = offset, threadIdx.x = chain
        const int64_t tt = t0 + threadIdx.y + i * kTR;
        v[i] = tt < P ? __ldcs(src + g * 32 * P + tt * 32 + threadIdx.x) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) tile[threadIdx.y + i * kTR][threadIdx.x] = v[i];
    __syncthreads();
    const int64_t t = t0 + threadIdx.x;
#pragma unroll
    for (int i = 0; i < R; ++i) {  // r = chain, threadIdx.x = offset
        const int64_t c = c0 + threadIdx.y + i * kTR;
        const int64_t x = c * P + t;
        if (c < nchains && t < P && x < N) {
            double y = tile[threadIdx.x][threadIdx.y + i * kTR];
            if (op == 2) y = log(y);
            __stcs(dst + x, y);
        }
    }
}

cudaError_t launch_to_t(const double *src, double *dst, int64_t N, int64_t P, int64_t nchains, int64_t nchp, int op,
                        cudaStream_t s, int64_t *launches, int *flags, double *mass, int allow_neg_inf) {
    dim3 grid((unsigned)((P + 31) / 32), (unsigned)(nchp / 32));
    k_to_t<<<grid, dim3(32, kTR), 0, s>>>(src, dst, N, P, nchains, op, flags, mass, allow_neg_inf);
    ++*launches;
    return cudaGetLastError();
}
cudaError_t launch_from_t(const double *src, double *dst, int64_t N, int64_t P, int64_t nchains, int64_t nchp, int op,
                          cudaStream_t s, int64_t *launches) {
    dim3 grid((unsigned)((P + 31) / 32), (unsigned)((nchains + 31) / 32));
    (void)nchp;
    k_from_t<<<grid, dim3(32, kTR), 0, s>>>(src, dst, N, P, nchains, op);
    ++*launches;
    return cudaGetLastError();
}

template <int NB, typename T>
static size_t ops_smem() {
    return (size_t)kWarpsPerCta * 2 * NB * 32 * (slab_s(NB) + 1) * sizeof(double);
}
template <int NB, int MODE>
static size_t apply_smem() {
    return (size_t)kWarpsPerCta * (2 * ApplyVecs<NB, MODE>::NV + 1) * 32 * (slab_s(NB) + 1) * sizeof(double);
}

template <int NB, typename T, int MODE, bool NEXT, bool FULL, bool PTS = false>
static void launch_apply_range(const Plan &p, int64_t cbeg, int64_t cend, cudaStream_t s, int64_t *launches) {
    if (cend <= cbeg) return;
    const size_t sm = apply_smem<NB, MODE>();
    smem_attr((const void *)k_chunk_apply<NB, T, MODE, NEXT, FULL, PTS>, sm);
    const int tpb = kWarpsPerCta * 32;
    const int64_t nb = (cend - cbeg + tpb - 1) / tpb;
    k_chunk_apply<NB, T, MODE, NEXT, FULL, PTS><<<(unsigned)nb, tpb, sm, s>>>(p, cbeg, cend);
    ++*launches;
}

// Full chains through the predicate-free kernel, the ragged last chain (or every chain when
// P is not a multiple of the slab length) through the general one.
template <int NB, int MODE, bool NEXT>
static void launch_apply_tm(const Plan &p, int64_t cbeg, int64_t cend, cudaStream_t s, int64_t *launches) {
    if (cend <= cbeg) return;
    const size_t sm = apply_smem<NB, MODE>();
    smem_attr((const void *)k_chunk_apply_tm<NB, MODE, NEXT>, sm);
    const int tpb = kWarpsPerCta * 32;
    const int64_t nb = (cend - cbeg + tpb - 1) / tpb;
    k_chunk_apply_tm<NB, MODE, NEXT><<<(unsigned)nb, tpb, sm, s>>>(p, cbeg, cend);
    ++*launches;
}

// Single-walk precision guard.  The inverse step B_{m+1} = D^-1 place_m^-1(B_m) subtracts; the
// rounding errors of the walked suffix states grow like their relative condition, which the forward
// (positive) recurrence never shrinks, so the error at a chain's END bounds the errors inside it.
// The end is checked where it matters, through the combine at the chain's last point m:
//   err = sum_S F_m[S] w_{|S|+1} |B_walked[S^c] - B_exact[S^c]|  <=  kSwGuardTol * J_exact[m],
// B_exact = the exact inclusive suffix carry of the next chain (the scan's car_bi); components that
// cannot reach J (tiny suffix states multiplied by small prefix states) cannot trip it.  For dual
// numbers (the cost) the tangent parts are checked the same way against the tangent of J.
// last: exact end state of the last chain (nullptr: e_empty); skip_last: do not check it.
template <int NB, typename T>
__global__ void k_sw_guard(const T *__restrict__ end, const T *__restrict__ cbi, const T *last, int skip_last,
                           Weights W, int64_t n, const int *stop, int *guard) {
    constexpr int M = 1 << NB;
    constexpr int K = sizeof(T) / sizeof(double);
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n || *stop) return;
    if (c + 1 >= n && skip_last) return;
    const double *bw = reinterpret_cast<const double *>(end + c * 2 * M);
    const double *fw = reinterpret_cast<const double *>(end + c * 2 * M + M);
    const double *be = c + 1 < n ? reinterpret_cast<const double *>(cbi + (c + 1) * M)
                                 : reinterpret_cast<const double *>(last);
    // value: J = sum F w B; tangent (duals): hatJ = sum (F' w + F w') B + F w B'
    double err[K], ref[K];
#pragma unroll
    for (int d = 0; d < K; ++d) err[d] = ref[d] = 0.0;
#pragma unroll
    for (int S = 0; S < M; ++S) {
        const int Sc = (M - 1) & ~S;
        const int a1 = __popc(S) + 1;
        const double a = W.w[a1] * fw[S * K];  // F w (value parts)
        const double bv = be ? be[Sc * K] : (Sc == 0 ? 1.0 : 0.0);
        const double dv = fabs(bw[Sc * K] - bv);
        err[0] += a * dv;
        ref[0] += a * bv;
        if constexpr (K == 2) {
            const double ad = W.w[a1] * fw[S * K + 1] + W.e[a1] * a;  // (F w)'
            const double bd = be ? be[Sc * K + 1] : 0.0;
            err[1] += a * fabs(bw[Sc * K + 1] - bd) + fabs(ad) * dv;
            ref[1] += ad * bv + a * bd;
        }
    }
    bool bad = false;
#pragma unroll
    for (int d = 0; d < K; ++d) bad |= !(err[d] <= kSwGuardTol * fabs(ref[d]));
    if (bad) atomicOr(guard, 1);
}

template <int NB, typename T>
static void launch_sw_guard(const Plan &p, cudaStream_t s, int64_t *launches) {
    constexpr int M = 1 << NB;
    const T *last = nullptr;
    int skip_last = 0;
    if (p.exch && p.rank + 1 < p.world) {
        if (p.rx_scan) skip_last = 1;  // the rank carry holds only the new parts (affine scan)
        else last = static_cast<const T *>(p.rank_car) + M;
    }
    k_sw_guard<NB, T><<<(unsigned)((p.nchunks + 255) / 256), 256, 0, s>>>(
        static_cast<const T *>(p.sw_end), static_cast<const T *>(p.car_bi), last, skip_last, p.W, p.nchunks, p.stop,
        p.guard);
    ++*launches;
}

template <int NB, int MODE>
static constexpr size_t sw_smem() {
    return (size_t)kWarpsPerCta * kSwStages * ApplyVecs<NB, MODE>::NV * kSwS * 32 * sizeof(double);
}

template <int NB, typename T, int MODE, bool NEXT, bool NXR = false>
static void launch_sw(const Plan &p, cudaStream_t s, int64_t *launches) {
    constexpr size_t sm = sw_smem<NB, MODE>();
    smem_attr((const void *)k_sw_apply<NB, T, MODE, NEXT, NXR>, sm);
    const int tpb = kWarpsPerCta * 32;
    const int64_t nb = (p.nchp + tpb - 1) / tpb;
    k_sw_apply<NB, T, MODE, NEXT, NXR><<<(unsigned)nb, tpb, sm, s>>>(p);
    ++*launches;
}

// Resident CTAs per SM of the single-walk update kernel (sizes the chain length in mmot_create).
int sw_blocks_per_sm(int NB) {
    int n = 0;
    const int tpb = kWarpsPerCta * 32;
    auto q = [&](auto kern, int nv, int) {
        const size_t sm = (size_t)kWarpsPerCta * kSwStages * nv * kSwS * 32 * sizeof(double);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, tpb, sm);
    };
    switch (NB) {
        case 1: q(k_sw_apply<1, double, MODE_UPD, true>, 2, slab_s(1)); break;
        case 2: q(k_sw_apply<2, double, MODE_UPD, true>, 3, slab_s(2)); break;
        case 3: q(k_sw_apply<3, double, MODE_UPD, true>, 4, slab_s(3)); break;
        case 4: q(k_sw_apply<4, double, MODE_UPD, true>, 5, slab_s(4)); break;
        default: n = 0;
    }
    cudaGetLastError();
    return n > 0 ? n : 2;
}

template <int NB, typename T, int MODE, bool NEXT = false>
static void launch_apply(const Plan &p, int64_t /*nb*/, int /*tpb*/, cudaStream_t s, int64_t *launches) {
    const bool full_ok = p.P % slab_s(NB) == 0;
    const int64_t nfull = full_ok ? p.N / p.P : 0;
    if constexpr (MODE == MODE_ALLRES) {
        // all-marginals residual pass (two-walk layout, uniform grids)
        launch_apply_range<NB, T, MODE, false, true>(p, 0, nfull, s, launches);
        launch_apply_range<NB, T, MODE, false, false>(p, nfull, p.nchunks, s, launches);
    } else {
        if (p.lam) {
            // non-uniform grid (two-walk contexts only; no fused next-update operators)
            if constexpr (!NEXT) {
                launch_apply_range<NB, T, MODE, false, true, true>(p, 0, nfull, s, launches);
                launch_apply_range<NB, T, MODE, false, false, true>(p, nfull, p.nchunks, s, launches);
            }
            return;
        }
        if (p.sw) {
            if constexpr (NB <= 4) {
                bool done = false;
                if constexpr (NEXT && MODE == MODE_UPD && sizeof(T) == sizeof(double) && NB >= 2) {
                    if (p.nxr) {
                        launch_sw<NB, T, MODE, false, true>(p, s, launches);
                        done = true;
                    }
                }
                if (!done) launch_sw<NB, T, MODE, NEXT>(p, s, launches);
                if (p.guard && p.sw_end) launch_sw_guard<NB, T>(p, s, launches);
            }
            return;
        }
        if constexpr (NB <= 3 && sizeof(T) == sizeof(double)) {
            if (p.P % (2 * sub_q(NB)) == 0 && p.P / (2 * sub_q(NB)) * 2 * (1 << NB) <= kTmemCols && !g_no_tmem) {
                launch_apply_tm<NB, MODE, NEXT>(p, 0, nfull, s, launches);
                launch_apply_range<NB, T, MODE, NEXT, false>(p, nfull, p.nchunks, s, launches);
                return;
            }
        }
        launch_apply_range<NB, T, MODE, NEXT, true>(p, 0, nfull, s, launches);
        launch_apply_range<NB, T, MODE, NEXT, false>(p, nfull, p.nchunks, s, launches);
    }
}

// ---------------------------------------------------------------------------------------
template <int NB, typename T>
__global__ void k_compose(const T *all, int world, int rank, T *car) {
    if (threadIdx.x == 0) compose_rank_carries<NB, T>(all, world, rank, car, car + (1 << NB));
}

template <int NB, typename T>
static cudaError_t product_nb(const Plan &p, int mode, cudaStream_t s, int64_t *launches, cudaEvent_t *ev,
                              bool with_ops, bool next) {
    const int tpb = kWarpsPerCta * 32;
    const int64_t nb = (p.nchunks + tpb - 1) / tpb;
    if (ev) cudaEventRecord(ev[0], s);
    if constexpr (NB >= 2 && NB <= 4 && sizeof(T) == sizeof(double)) {
        if (p.rx_scan && mode == MODE_UPD) {
            if (ev) cudaEventRecord(ev[1], s);
            launch_rx_scan<NB>(p, s, launches);
            if (ev) cudaEventRecord(ev[2], s);
            launch_apply<NB, T, MODE_UPD, true>(p, nb, tpb, s, launches);
            if (ev) cudaEventRecord(ev[3], s);
            return cudaGetLastError();
        }
    }
    if (with_ops && p.sw) {
        if constexpr (NB <= 4) {
            constexpr size_t sm = (size_t)kWarpsPerCta * kSwStages * NB * kSwS * 32 * sizeof(double);
            smem_attr((const void *)k_sw_ops<NB, T>, sm);
            k_sw_ops<NB, T><<<(unsigned)((p.nchp + tpb - 1) / tpb), tpb, sm, s>>>(p);
            ++*launches;
        }
    } else if (with_ops && NB == 5 && sizeof(T) == sizeof(double) && !p.lam) {
        if constexpr (NB == 5 && sizeof(T) == sizeof(double)) {
            const unsigned g = (unsigned)((p.nchunks + kOpsSplitChunks - 1) / kOpsSplitChunks);
            if (mode == MODE_ALLRES) k_chunk_ops_split<NB, true><<<g, 2 * kOpsSplitChunks, 0, s>>>(p);
            else k_chunk_ops_split<NB><<<g, 2 * kOpsSplitChunks, 0, s>>>(p);
            ++*launches;
        }
    } else if (with_ops) {
        const size_t sm = ops_smem<NB, T>();
        smem_attr((const void *)k_chunk_ops<NB, T>, sm);
        smem_attr((const void *)k_chunk_ops<NB, T, true>, sm);
        if (mode == MODE_ALLRES) {
            if constexpr (sizeof(T) == sizeof(double)) {
                smem_attr((const void *)k_chunk_ops<NB, T, false, true>, sm);
                k_chunk_ops<NB, T, false, true><<<(unsigned)nb, tpb, sm, s>>>(p);
            }
        } else if (p.lam) {
            k_chunk_ops<NB, T, true><<<(unsigned)nb, tpb, sm, s>>>(p);
        } else {
            k_chunk_ops<NB, T><<<(unsigned)nb, tpb, sm, s>>>(p);
        }
        ++*launches;
    }
    if (ev) cudaEventRecord(ev[1], s);
    constexpr bool kWarpScan = NB <= 3 && sizeof(T) == sizeof(double);
    const int top = p.nlev - 1;
    // up-sweep
    for (int i = 0; i + 1 < p.nlev; ++i) {
        const int64_t ng = p.nlev_n[i + 1];
        if constexpr (kWarpScan) {
            dim3 grid((unsigned)((ng + 3) / 4), 2);
            k_ops_reduce_w<NB><<<grid, 128, 0, s>>>(static_cast<const double *>(p.ops_f[i]),
                                                     static_cast<const double *>(p.ops_b[i]),
                                                     static_cast<double *>(p.ops_f[i + 1]),
                                                     static_cast<double *>(p.ops_b[i + 1]), p.nlev_n[i], p.stop);
            ++*launches;
            continue;
        }
        if constexpr (NB >= 4 && sizeof(T) == sizeof(double)) {
            k_ops_reduce_t<NB><<<dim3((unsigned)ng, 2), 128, 0, s>>>(
                reinterpret_cast<const double *>(p.ops_f[i]), reinterpret_cast<const double *>(p.ops_b[i]),
                reinterpret_cast<double *>(p.ops_f[i + 1]), reinterpret_cast<double *>(p.ops_b[i + 1]), p.nlev_n[i],
                p.stop);
            ++*launches;
            continue;
        }
        if constexpr (NB >= 4) {
            k_ops_reduce_c<NB, T><<<dim3((unsigned)ng, 2), 128, 0, s>>>(
                static_cast<const T *>(p.ops_f[i]), static_cast<const T *>(p.ops_b[i]), static_cast<T *>(p.ops_f[i + 1]),
                static_cast<T *>(p.ops_b[i + 1]), p.nlev_n[i], p.stop);
            ++*launches;
            continue;
        }
        dim3 grid((unsigned)((ng + 63) / 64), 2);
        k_ops_reduce<NB, T><<<grid, 64, 0, s>>>(static_cast<const T *>(p.ops_f[i]), static_cast<const T *>(p.ops_b[i]),
                                               static_cast<T *>(p.ops_f[i + 1]), static_cast<T *>(p.ops_b[i + 1]),
                                               p.nlev_n[i], p.stop);
        ++*launches;
    }
    // sharded contexts: whole-shard operators (top level reduced to one), exchanged between the
    // ranks, composed into the carries entering this shard (compose_rank_carries)
    if (p.exch) {
        if constexpr (kWarpScan) {
            k_ops_reduce_w<NB><<<dim3(1, 2), 128, 0, s>>>(static_cast<const double *>(p.ops_f[top]),
                                                          static_cast<const double *>(p.ops_b[top]),
                                                          static_cast<double *>(p.agg_send),
                                                          static_cast<double *>(p.agg_send) + OpShape<NB>::SZ,
                                                          p.nlev_n[top], p.stop);
        } else if constexpr (NB >= 4) {
            k_ops_reduce_c<NB, T><<<dim3(1, 2), 128, 0, s>>>(static_cast<const T *>(p.ops_f[top]),
                                                            static_cast<const T *>(p.ops_b[top]),
                                                            static_cast<T *>(p.agg_send),
                                                            static_cast<T *>(p.agg_send) + OpShape<NB>::SZ,
                                                            p.nlev_n[top], p.stop);
        } else {
            k_ops_reduce<NB, T><<<dim3(1, 2), 64, 0, s>>>(static_cast<const T *>(p.ops_f[top]),
                                                         static_cast<const T *>(p.ops_b[top]),
                                                         static_cast<T *>(p.agg_send),
                                                         static_cast<T *>(p.agg_send) + OpShape<NB>::SZ,
                                                         p.nlev_n[top], p.stop);
        }
        ++*launches;
        p.exch(p.exch_ctx, 2 * (size_t)OpShape<NB>::SZ * (sizeof(T) / sizeof(double)), s);
        k_compose<NB, T><<<1, 1, 0, s>>>(static_cast<const T *>(p.agg_all), p.world, p.rank,
                                         static_cast<T *>(p.rank_car));
        ++*launches;
    }
    // down-sweep
    for (int i = p.nlev - 1; i >= 0; --i) {
        const int64_t ng = (p.nlev_n[i] + group_of(NB) - 1) / group_of(NB);
        dim3 grid((unsigned)((ng + 63) / 64), 2);
        const T *gf = i + 1 < p.nlev ? static_cast<const T *>(p.car_f[i + 1])
                                     : (p.exch ? static_cast<const T *>(p.rank_car) : nullptr);
        const T *gb = i + 1 < p.nlev ? static_cast<const T *>(p.car_b[i + 1])
                                     : (p.exch ? static_cast<const T *>(p.rank_car) + (1 << NB) : nullptr);
        if constexpr (kWarpScan) {
            dim3 gridw((unsigned)((ng + 3) / 4), 2);
            k_ops_down_w<NB><<<gridw, 128, 0, s>>>(static_cast<const double *>(p.ops_f[i]),
                                                    static_cast<const double *>(p.ops_b[i]),
                                                    reinterpret_cast<const double *>(gf),
                                                    reinterpret_cast<const double *>(gb),
                                                    static_cast<double *>(p.car_f[i]), static_cast<double *>(p.car_b[i]),
                                                    p.nlev_n[i], p.stop,
                                                    i == 0 && p.sw ? static_cast<double *>(p.car_bi) : nullptr);
            ++*launches;
            continue;
        }
        if constexpr (NB >= 4 && sizeof(T) == sizeof(double)) {
            k_ops_down_cw<NB><<<dim3((unsigned)((ng + 1) / 2), 2), 64, 0, s>>>(
                reinterpret_cast<const double *>(p.ops_f[i]), reinterpret_cast<const double *>(p.ops_b[i]),
                reinterpret_cast<const double *>(gf), reinterpret_cast<const double *>(gb),
                reinterpret_cast<double *>(p.car_f[i]), reinterpret_cast<double *>(p.car_b[i]), p.nlev_n[i], p.stop,
                i == 0 && p.sw ? reinterpret_cast<double *>(p.car_bi) : nullptr);
            ++*launches;
            continue;
        }
        if constexpr (NB >= 4) {
            k_ops_down_c<NB, T><<<dim3((unsigned)ng, 2), 64, 0, s>>>(
                static_cast<const T *>(p.ops_f[i]), static_cast<const T *>(p.ops_b[i]), gf, gb, static_cast<T *>(p.car_f[i]),
                static_cast<T *>(p.car_b[i]), p.nlev_n[i], p.stop, i == 0 && p.sw ? static_cast<T *>(p.car_bi) : nullptr);
            ++*launches;
            continue;
        }
        k_ops_down<NB, T><<<grid, 64, 0, s>>>(static_cast<const T *>(p.ops_f[i]), static_cast<const T *>(p.ops_b[i]),
                                             gf, gb, static_cast<T *>(p.car_f[i]), static_cast<T *>(p.car_b[i]),
                                             p.nlev_n[i], p.stop, i == 0 && p.sw ? static_cast<T *>(p.car_bi) : nullptr);
        ++*launches;
    }
    if (ev) cudaEventRecord(ev[2], s);
    switch (mode) {
        case MODE_MARG: launch_apply<NB, T, MODE_MARG>(p, nb, tpb, s, launches); break;
        case MODE_UPD:
            if (next && NB <= 4 && !p.lam) {
                if constexpr (sizeof(T) == sizeof(double) && NB <= 4)
                    launch_apply<NB, T, MODE_UPD, true>(p, nb, tpb, s, launches);
            } else {
                launch_apply<NB, T, MODE_UPD>(p, nb, tpb, s, launches);
            }
            break;
        case MODE_RES: launch_apply<NB, T, MODE_RES>(p, nb, tpb, s, launches); break;
        case MODE_ALLRES:
            if constexpr (sizeof(T) == sizeof(double)) launch_apply<NB, T, MODE_ALLRES>(p, nb, tpb, s, launches);
            break;
        default: launch_apply<NB, T, MODE_COST>(p, nb, tpb, s, launches); break;
    }
    if (ev) cudaEventRecord(ev[3], s);
    return cudaGetLastError();
}

cudaError_t launch_product(const Plan &p, int mode, cudaStream_t s, int64_t *launches, cudaEvent_t *ev,
                           bool with_ops, bool next) {
    const bool dual = mode == MODE_COST;
    if (p.ls && p.NB == 5 && (mode == MODE_UPD || mode == MODE_MARG || mode == MODE_RES)) {
        if (ev) cudaEventRecord(ev[0], s);
        if (ev) cudaEventRecord(ev[1], s);
        if (ev) cudaEventRecord(ev[2], s);
        cudaError_t e = launch_ls_product(p, *p.ls, mode, s, launches);
        if (ev) cudaEventRecord(ev[3], s);
        return e;
    }
    switch (p.NB) {
        case 1: return dual ? product_nb<1, Dual>(p, mode, s, launches, ev, with_ops, next) : product_nb<1, double>(p, mode, s, launches, ev, with_ops, next);
        case 2: return dual ? product_nb<2, Dual>(p, mode, s, launches, ev, with_ops, next) : product_nb<2, double>(p, mode, s, launches, ev, with_ops, next);
        case 3: return dual ? product_nb<3, Dual>(p, mode, s, launches, ev, with_ops, next) : product_nb<3, double>(p, mode, s, launches, ev, with_ops, next);
        case 4: return dual ? product_nb<4, Dual>(p, mode, s, launches, ev, with_ops, next) : product_nb<4, double>(p, mode, s, launches, ev, with_ops, next);
        case 5: return dual ? product_nb<5, Dual>(p, mode, s, launches, ev, with_ops, next) : product_nb<5, double>(p, mode, s, launches, ev, with_ops, next);
        default: return cudaErrorInvalidValue;
    }
}

// ---------------------------------------------------------------------------------------
// Small kernels.
// ---------------------------------------------------------------------------------------
void smem_attr(const void *func, size_t bytes) {
    static std::mutex mu;
    static std::set<std::tuple<const void *, int, size_t>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (done.insert(std::make_tuple(func, dev, bytes)).second)
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// In-process group reduction (virtual shards): out[i] = op over r of src[r][i].
__global__ void k_vreduce(VPtrs src, int world, int n, int op, void *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (op == 0) {
        double acc = 0.0;
        for (int r = 0; r < world; ++r) acc += static_cast<const double *>(src.p[r])[i];
        static_cast<double *>(out)[i] = acc;
    } else {
        int acc = static_cast<const int *>(src.p[0])[i];
        for (int r = 1; r < world; ++r) acc = max(acc, static_cast<const int *>(src.p[r])[i]);
        static_cast<int *>(out)[i] = acc;
    }
}

cudaError_t launch_vreduce(const VPtrs &src, int world, int n, int op, void *out, cudaStream_t s, int64_t *launches) {
    k_vreduce<<<(n + 127) / 128, 128, 0, s>>>(src, world, n, op, out);
    ++*launches;
    return cudaGetLastError();
}
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

// fp32 I/O contexts (MMOT_F32): widen the caller's float marginals, narrow float outputs.
__global__ void k_f32_to_f64(const float *__restrict__ in, double *__restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
__global__ void k_f64_to_f32(const double *__restrict__ in, float *__restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}
cudaError_t launch_convert(const void *in, void *out, int64_t n, int to_f64, cudaStream_t s, int64_t *launches) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (to_f64) k_f32_to_f64<<<grid, 256, 0, s>>>(static_cast<const float *>(in), static_cast<double *>(out), n);
    else k_f64_to_f32<<<grid, 256, 0, s>>>(static_cast<const double *>(in), static_cast<float *>(out), n);
    ++*launches;
    return cudaGetLastError();
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

__global__ void k_resid_finish(double *acc, double tol, const int *sweep, double *res_out, int *iters_done,
                               int *converged, int *stop) {
    if (*stop) return;
    const double r = *acc;
    *res_out = r;
    *iters_done = *sweep;
    if (r <= tol) {
        *converged = 1;
        *stop = 1;
    }
}

cudaError_t launch_resid_finish(double *acc, double tol, const int *sweep, double *res_out, int *iters_done,
                                int *converged, int *stop, cudaStream_t s, int64_t *launches) {
    k_resid_finish<<<1, 1, 0, s>>>(acc, tol, sweep, res_out, iters_done, converged, stop);
    ++*launches;
    return cudaGetLastError();
}

// End of a sweep: unless the solve has stopped, count it (sweep = completed sweeps, read by the
// residual check and by raise_status) and report it.
__global__ void k_sweep_done(int *sweep, int *iters_done, const int *stop) {
    if (*stop) return;
    const int t = *sweep + 1;
    *sweep = t;
    *iters_done = t;
}
cudaError_t launch_sweep_done(int *sweep, int *iters_done, const int *stop, cudaStream_t s, int64_t *launches) {
    k_sweep_done<<<1, 1, 0, s>>>(sweep, iters_done, stop);
    ++*launches;
    return cudaGetLastError();
}

// Device-resident Sinkhorn loop (CUDA graph with a conditional WHILE node, api.cu): the last node of
// the loop body counts the periods and keeps looping while periods remain and nothing stopped.
__global__ void k_loop_cond(cudaGraphConditionalHandle h, int *done, const int *n, const int *stop) {
    const int d = *done + 1;
    *done = d;
    cudaGraphSetConditional(h, (d < *n && !*(volatile const int *)stop) ? 1u : 0u);
}
cudaError_t launch_loop_cond(cudaGraphConditionalHandle h, int *done, const int *n, const int *stop, cudaStream_t s,
                             int64_t *launches) {
    k_loop_cond<<<1, 1, 0, s>>>(h, done, n, stop);
    ++*launches;
    return cudaGetLastError();
}
}  // namespace mmot
