// dp.cuh -- device building blocks of the O(N) tensor-vector product (arXiv 2405.19246).
//
// The paper splits the index set into the l! order regions D_p,
// makes the exponent linear inside each region and evaluates every region by
// nested prefix/suffix sums computed with first-order recurrences ("separated summations
// and dynamic programming").  On the GPU we use the equivalent
// edge form of the same exponent:
//
//     E(i) = sum_{p<q} |i_p - i_q| = sum_{x=0}^{N-2} a_x (l - a_x),
//     a_x  = #{ indices at or left of grid point x }.
//
// Every grid edge with a indices on its left contributes w_a = lambda^{a(l-a)}, so the l!
// region chains collapse into one left-to-right recurrence over the 2^{l-1} subsets S of
// the bound marginals B = {1..l}\{k} ("which bound marginals are already placed"):
//
//     F_x[S] = sum_{T subset S} w_{|S\T|} F_{x-1}[S\T] prod_{q in T} phi_q[x]     (prefix)
//     B_x[R] = sum_{T subset R} w_{|R\T|} B_{x+1}[R\T] prod_{q in T} phi_q[x]     (suffix)
//     J_k[m] = sum_{S subset B} F_m[S] * w_{|S|+1} * B_{m+1}[B\S]                 (combine)
//
// Each state is a first-order constant-decay recurrence s[x] = w s[x-1] + v[x] (north_star)
// whose input v comes from lower subset levels.  A step is "diag" (multiply by w_{|S|},
// the edge crossed) followed by "place" (in-place rank-1 updates, one per bound marginal,
// which also realises ties i_p = i_q).
//
// Chunk operators.  The state after a chunk is linear in the state before it.  Because
// the edge weight only depends on the COUNT of indices already placed, the operator has
// the form  Op(F)[S] = sum_{U subset S} F[U] * G_{|U|}[S\U],  where G_c is the chunk DP
// started from the empty set with weights shifted by c (w_{c+|V|}).  Only entries with
// |V| <= NB - c are ever used.  Operators compose in the same form, which gives the
// parallel (hierarchical) scan over chunks.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace mmot {

constexpr int kMaxL = 6;

// popcount; non-recursive and force-inlined so that it folds to a constant inside the
// fully unrolled subset loops (a recursive constexpr is emitted as a real CALL otherwise).
__host__ __device__ __forceinline__ constexpr int pc(int x) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) c += (x >> i) & 1;
    return c;
}

// ---------------------------------------------------------------------------------------
// Scalar types: plain double, and a dual number (value, d/dlog(lambda)) for the cost.
// With w_a = lambda^{e_a}, dw_a/dlog(lambda) = e_a w_a, so carrying duals through the
// same scans yields hatJ = sum_i E(i) lambda^{E(i)} prod phi.
// ---------------------------------------------------------------------------------------
struct Dual {
    double v, d;
};

__host__ __device__ __forceinline__ double zero_of(double) { return 0.0; }
__device__ __forceinline__ Dual zero_of(Dual) { return Dual{0.0, 0.0}; }
__host__ __device__ __forceinline__ double one_of(double) { return 1.0; }
__device__ __forceinline__ Dual one_of(Dual) { return Dual{1.0, 0.0}; }

// a * b
__host__ __device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ Dual mul(Dual a, Dual b) { return Dual{a.v * b.v, fma(a.d, b.v, a.v * b.d)}; }
// acc + a * b
__host__ __device__ __forceinline__ double mad(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ Dual mad(Dual a, Dual b, Dual acc) {
    return Dual{fma(a.v, b.v, acc.v), fma(a.d, b.v, fma(a.v, b.d, acc.d))};
}
// acc + f * b  with a plain scalar f (scaling vector entry)
__device__ __forceinline__ double mads(double f, double b, double acc) { return fma(f, b, acc); }
__device__ __forceinline__ Dual mads(double f, Dual b, Dual acc) { return Dual{fma(f, b.v, acc.v), fma(f, b.d, acc.d)}; }

__device__ __forceinline__ Dual operator+(Dual a, Dual b) { return Dual{a.v + b.v, a.d + b.d}; }

__device__ __forceinline__ double value_of(double a) { return a; }
__device__ __forceinline__ double value_of(Dual a) { return a.v; }

// Edge weight w_a as scalar type T (dual part e_a w_a).
struct Weights {
    double w[kMaxL + 1];  // w_a = exp(-a(l-a) h / eta), a = 0..l
    double e[kMaxL + 1];  // e_a = a(l-a)
};
__device__ __forceinline__ void load_weight(double &o, const Weights &W, int a) { o = W.w[a]; }
__device__ __forceinline__ void load_weight(Dual &o, const Weights &W, int a) { o = Dual{W.w[a], W.e[a] * W.w[a]}; }

// ---------------------------------------------------------------------------------------
// One grid point of the recurrence.  `wc[a]` = w_{c+a}; states S with popcount > LIMIT are
// not needed (operators) and are skipped at compile time.
// ---------------------------------------------------------------------------------------
// W0ONE: wc[0] is w_0 = lambda^0 = 1 exactly, so the empty-set state needs no multiply.
template <int NB, typename T, bool W0ONE = false>
__device__ __forceinline__ void dp_diag(T (&st)[1 << NB], const T *wc, int limit = NB) {
#pragma unroll
    for (int S = W0ONE ? 1 : 0; S < (1 << NB); ++S)
        if (pc(S) <= limit) st[S] = mul(wc[pc(S)], st[S]);
}

template <int NB, typename T>
__device__ __forceinline__ void dp_place(T (&st)[1 << NB], const double (&f)[NB > 0 ? NB : 1], int limit = NB) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
        for (int S = (1 << NB) - 1; S >= 0; --S)
            if ((S >> b) & 1)
                if (pc(S) <= limit) st[S] = mads(f[b], st[S ^ (1 << b)], st[S]);
    }
}

// Inverse of dp_place: st <- place_x^{-1}(st).  place_x = prod_q (I + phi_q[x] E_q) with
// commuting nilpotent E_q (E_q^2 = 0), so place_x^{-1} = prod_q (I - phi_q[x] E_q).
template <int NB, typename T>
__device__ __forceinline__ void dp_unplace(T (&st)[1 << NB], const double (&f)[NB > 0 ? NB : 1]) {
#pragma unroll
    for (int b = NB - 1; b >= 0; --b) {
#pragma unroll
        for (int S = 0; S < (1 << NB); ++S)
            if ((S >> b) & 1) st[S] = mads(-f[b], st[S ^ (1 << b)], st[S]);
    }
}

// st[S] *= winv[|S|] for S != {} (winv[0] = 1/w_0 = 1).
template <int NB, typename T>
__device__ __forceinline__ void dp_diag_inv(T (&st)[1 << NB], const T *winv) {
#pragma unroll
    for (int S = 1; S < (1 << NB); ++S) st[S] = mul(winv[pc(S)], st[S]);
}

// Per-level diag in a frame scaled by w_1 per grid step (single-walk kernels, fp64): st[S] *= c[|S|]
// except for the levels whose multiplier is exactly 1 (|S| = 1 and |S| = NB: w_{l-1} = w_1, l = NB+1),
// which are skipped at compile time.  DESIGN.md §5 (scaled frames).
template <int NB>
__device__ __forceinline__ void dp_diag_lvl(double (&st)[1 << NB], const double (&c)[NB + 2]) {
#pragma unroll
    for (int S = 0; S < (1 << NB); ++S) {
        const int a = pc(S);
        if (a != 1 && a != NB) st[S] *= c[a];
    }
}

// Operator storage: G[c][S], c = 0..NB, S = 0..2^NB-1 (entries with pc(S) > NB-c unused).
template <int NB>
struct OpShape {
    static constexpr int M = 1 << NB;
    static constexpr int SZ = (NB + 1) * M;
};

template <int NB, typename T>
__device__ __forceinline__ void op_identity(T (&G)[NB + 1][1 << NB]) {
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int S = 0; S < (1 << NB); ++S) G[c][S] = (S == 0) ? one_of(T{}) : zero_of(T{});
}

// ---------------------------------------------------------------------------------------
// One walk for both chain operators (prefix/suffix duality).
//
// Let Gt_c be the chain DP from e_{} with weights w_{c+|V|}, WITHOUT the diag of its first
// grid point (the edge entering the chain).  Then the prefix operator is G_c = w_c Gt_c and,
// because the edge weight of a suffix walk counts the indices to the RIGHT of an edge
// (|V| - #left) and w_a = w_{l-a}, the suffix operator is
//     R_c[V] = w_c * Gt_{l-c-|V|}[V]                     (l = NB+1; Gt_l[{}] = 1)
// (exact identity of the two sums; pinned by the GPU parity tests and DESIGN.md §1).
// Gt is needed on the extended range c + |V| <= l, slices c = 0..NB: one walk of ~2/3 the
// cost of walking the prefix and the suffix operators separately.
// ---------------------------------------------------------------------------------------
template <int NB, typename T>
__device__ __forceinline__ void opx_identity(T (&G)[NB + 1][1 << NB]) {
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int S = 0; S < (1 << NB); ++S) G[c][S] = (S == 0) ? one_of(T{}) : zero_of(T{});
}

// wt[a] = w_a, a = 0..NB+1 (w_{NB+1} = w_l = 1 and w_0 = 1 are not multiplied).
template <int NB, typename T>
__device__ __forceinline__ void opx_step(T (&G)[NB + 1][1 << NB], const T *wt, const double (&f)[NB > 0 ? NB : 1],
                                         bool skip_diag) {
    constexpr int L = NB + 1;
    if (!skip_diag) {
#pragma unroll
        for (int c = 0; c <= NB; ++c)
#pragma unroll
            for (int V = 0; V < (1 << NB); ++V) {
                const int a = c + pc(V);
                if (a < L && a > 0) G[c][V] = mul(wt[a], G[c][V]);
            }
    }
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int V = (1 << NB) - 1; V >= 0; --V)
                if (((V >> b) & 1) && c + pc(V) <= L) G[c][V] = mads(f[b], G[c][V ^ (1 << b)], G[c][V]);
}

// Store the prefix operator (w_c Gt_c) and the suffix operator (w_c Gt_{l-c-|V|}) in op_store
// layout.  LW = l, the marginal count of the weights w_a = lambda^{a(l-a)} = w_{l-a}: NB + 1 for a
// product's bound set (NB = l - 1), NB for the DP over all l scalings (MODE_ALLRES, NB = l).
template <int NB, typename T, int LW = NB + 1>
__device__ __forceinline__ void opx_store(const T (&G)[NB + 1][1 << NB], const T *wt, T *pf, T *pb) {
    constexpr int M = 1 << NB;
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int V = 0; V < M; ++V)
            if (c + pc(V) <= NB) {
                const int cp = LW - c - pc(V);
                pf[c * M + V] = c == 0 ? G[0][V] : mul(wt[c], G[c][V]);
                const T r = cp > NB ? one_of(T{}) : G[cp][V];
                pb[c * M + V] = c == 0 ? r : mul(wt[c], r);
            }
}

// Chain operators under per-edge weights: prefix operator w_c(entry edge) Gt_c, suffix operator
// w_c(exit edge) Gt_{l-c-|V|} (the duality of opx_store with the two boundary edges made explicit:
// the chain's internal edges carry the same exponents in both, DESIGN.md §2 A20).
template <int NB, typename T>
__device__ __forceinline__ void opx_store_pts(const T (&G)[NB + 1][1 << NB], const T *win, const T *wout, T *pf, T *pb) {
    constexpr int M = 1 << NB;
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int V = 0; V < M; ++V)
            if (c + pc(V) <= NB) {
                const int cp = NB + 1 - c - pc(V);
                pf[c * M + V] = c == 0 ? G[0][V] : mul(win[c], G[c][V]);
                const T r = cp > NB ? one_of(T{}) : G[cp][V];
                pb[c * M + V] = c == 0 ? r : mul(wout[c], r);
            }
}

// out = Op(in):  out[S] = sum_{U subset S} in[U] * G[|U|][S\U]
template <int NB, typename T>
__host__ __device__ __forceinline__ void op_apply(const T (&G)[NB + 1][1 << NB], const T (&in)[1 << NB], T (&out)[1 << NB]) {
#pragma unroll
    for (int S = 0; S < (1 << NB); ++S) {
        T acc = zero_of(T{});
#pragma unroll
        for (int U = 0; U < (1 << NB); ++U)
            if ((U & S) == U) acc = mad(in[U], G[pc(U)][S ^ U], acc);
        out[S] = acc;
    }
}

// C = B o A (A applied first):  C_c[V] = sum_{U subset V} A_c[U] * B_{c+|U|}[V\U]
template <int NB, typename T>
__device__ __forceinline__ void op_compose(const T (&A)[NB + 1][1 << NB], const T (&B)[NB + 1][1 << NB],
                                           T (&C)[NB + 1][1 << NB]) {
#pragma unroll
    for (int c = 0; c <= NB; ++c) {
#pragma unroll
        for (int V = 0; V < (1 << NB); ++V) {
            if (pc(V) > NB - c) { C[c][V] = zero_of(T{}); continue; }
            T acc = zero_of(T{});
#pragma unroll
            for (int U = 0; U < (1 << NB); ++U)
                if ((U & V) == U) acc = mad(A[c][U], B[c + pc(U)][V ^ U], acc);
            C[c][V] = acc;
        }
    }
}

template <int NB, typename T>
__host__ __device__ __forceinline__ void op_load(T (&G)[NB + 1][1 << NB], const T *p) {
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int S = 0; S < (1 << NB); ++S)
            if (pc(S) <= NB - c) G[c][S] = p[c * (1 << NB) + S];
            else G[c][S] = zero_of(T{});
}

template <int NB, typename T>
__device__ __forceinline__ void op_store(const T (&G)[NB + 1][1 << NB], T *p) {
#pragma unroll
    for (int c = 0; c <= NB; ++c)
#pragma unroll
        for (int S = 0; S < (1 << NB); ++S)
            if (pc(S) <= NB - c) p[c * (1 << NB) + S] = G[c][S];
}

template <int NB, typename T>
__device__ __forceinline__ void vec_load(T (&v)[1 << NB], const T *p) {
#pragma unroll
    for (int S = 0; S < (1 << NB); ++S) v[S] = p[S];
}
template <int NB, typename T>
__device__ __forceinline__ void vec_store(const T (&v)[1 << NB], T *p) {
#pragma unroll
    for (int S = 0; S < (1 << NB); ++S) p[S] = v[S];
}
template <int NB, typename T>
__host__ __device__ __forceinline__ void vec_unit(T (&v)[1 << NB]) {
#pragma unroll
    for (int S = 0; S < (1 << NB); ++S) v[S] = (S == 0) ? one_of(T{}) : zero_of(T{});
}

// ---------------------------------------------------------------------------------------
// Multi-GPU (sharded contexts): rank g owns a contiguous grid chunk; after the scan every rank
// holds its whole-chunk prefix operator Gg and suffix operator Rg (the composition of all its
// chain operators).  The carry entering rank g from the left is G_{g-1} o ... o G_0 (e_{}),
// the one entering from the right is R_{g+1} o ... o R_{G-1} (e_{}).  `all` holds the gathered
// [world][2][SZ] operators (prefix, suffix) in op_store layout.  Same code on host and device.
template <int NB, typename T>
__host__ __device__ inline void compose_rank_carries(const T *all, int world, int rank, T *fin, T *bin) {
    constexpr int M = 1 << NB;
    constexpr int SZ = (NB + 1) * M;
    T cur[M], nxt[M], G[NB + 1][M];
    vec_unit<NB, T>(cur);
    for (int r = 0; r < rank; ++r) {
        op_load<NB, T>(G, all + ((size_t)r * 2 + 0) * SZ);
        op_apply<NB, T>(G, cur, nxt);
        for (int S = 0; S < M; ++S) cur[S] = nxt[S];
    }
    for (int S = 0; S < M; ++S) fin[S] = cur[S];
    vec_unit<NB, T>(cur);
    for (int r = world - 1; r > rank; --r) {
        op_load<NB, T>(G, all + ((size_t)r * 2 + 1) * SZ);
        op_apply<NB, T>(G, cur, nxt);
        for (int S = 0; S < M; ++S) cur[S] = nxt[S];
    }
    for (int S = 0; S < M; ++S) bin[S] = cur[S];
}

// ---------------------------------------------------------------------------------------
// Restricted next-update scan (single-walk Sinkhorn updates).  Update k+1's bound slots are
// (slot 1..NB-1 of update k, then the new phi_k).  Its states S' = U (U over the NB-1 "old"
// slots) equal update k's states U << 1 exactly (same marginals, unchanged vectors), so only the
// "new part" S' = U + {new} needs a scan, and it is affine in the carry:
//   prefix  y_out = A'(y_in) + L,   suffix  z_start = A''(z_end) + M,
// where A', A'' are operators of the (NB-1)-marginal DP on the old slots with shifts c = 1..NB
// (entries G_c[V], c + |V| <= NB; A'' from the same walk by the prefix/suffix duality), and
// L, M are accumulated along update k's walk from its exact states.
// Element layout (SZE = (NB+1) * MO doubles): A[c-1][V] at (c-1)*MO + V, offset at NB*MO + U.
// ---------------------------------------------------------------------------------------
template <int NB>
struct Rx {
    static constexpr int NO = NB - 1;
    static constexpr int MO = 1 << (NB - 1);
    static constexpr int SZE = (NB + 1) * MO;
};

// L <- place_old(D L) + o * F_old   (F = update k's prefix state AFTER this point's step)
template <int NB>
__device__ __forceinline__ void rx_L_step(double (&L)[Rx<NB>::MO], const double *wt, const double (&f)[NB],
                                          double o, const double (&F)[1 << NB]) {
    constexpr int MO = Rx<NB>::MO;
#pragma unroll
    for (int U = 0; U < MO; ++U) L[U] *= wt[pc(U) + 1];
#pragma unroll
    for (int j = 0; j < NB - 1; ++j)
#pragma unroll
        for (int U = MO - 1; U >= 0; --U)
            if ((U >> j) & 1) L[U] = fma(f[j + 1], L[U ^ (1 << j)], L[U]);
#pragma unroll
    for (int U = 0; U < MO; ++U) L[U] = fma(o, F[U << 1], L[U]);
}

// rx_L_step on L scaled by w_1^{-t} (the prefix frame of the scaled single walk, F~ = F w_1^{-t}):
// L~ <- place_old(D' L~) + o F~_old with D' = D / w_1 (wr[a] = w_a / w_1; levels a = |U| + 1 in
// {1, NB} need no multiply).  The caller unscales once at the chain end.
template <int NB>
__device__ __forceinline__ void rx_L_step_scl(double (&L)[Rx<NB>::MO], const double *wr, const double (&f)[NB],
                                              double o, const double (&F)[1 << NB]) {
    constexpr int MO = Rx<NB>::MO;
#pragma unroll
    for (int U = 0; U < MO; ++U) {
        const int a = pc(U) + 1;
        if (a != 1 && a != NB) L[U] *= wr[a];
    }
#pragma unroll
    for (int j = 0; j < NB - 1; ++j)
#pragma unroll
        for (int U = MO - 1; U >= 0; --U)
            if ((U >> j) & 1) L[U] = fma(f[j + 1], L[U ^ (1 << j)], L[U]);
#pragma unroll
    for (int U = 0; U < MO; ++U) L[U] = fma(o, F[U << 1], L[U]);
}

// Running restricted operator Gr[c-1][V] (c = 1..NB, V over old slots, c+|V| <= NB); the diag
// of the chain's first point is skipped (G~ convention of opx_*).
template <int NB>
__device__ __forceinline__ void rx_G_step(double (&G)[NB][Rx<NB>::MO], const double *wt, const double (&f)[NB], bool skip) {
    constexpr int MO = Rx<NB>::MO;
    if (!skip) {
#pragma unroll
        for (int c = 1; c <= NB; ++c)
#pragma unroll
            for (int V = 0; V < MO; ++V)
                if (c + pc(V) <= NB) G[c - 1][V] *= wt[c + pc(V)];
    }
#pragma unroll
    for (int c = 1; c <= NB; ++c)
#pragma unroll
        for (int j = 0; j < NB - 1; ++j)
#pragma unroll
            for (int V = MO - 1; V >= 0; --V)
                if (((V >> j) & 1) && c + pc(V) <= NB) G[c - 1][V] = fma(f[j + 1], G[c - 1][V ^ (1 << j)], G[c - 1][V]);
}

// rx_G_step on the running operator scaled by s_t = w_1^t (t = diag steps applied so far): an
// entry with c + |V| = a is multiplied by w_a / w_1, so entries with a in {1, l-1} (w_a = w_1)
// need no multiply.  The caller keeps s_t (one multiply per point) and unscales at the uses
// (rx_M_acc with o * s_t, rx_store with the entries times s_t).  wr[a] = w_a / w_1.
template <int NB>
__device__ __forceinline__ void rx_G_step_scaled(double (&G)[NB][Rx<NB>::MO], const double *wr, const double (&f)[NB],
                                                 bool skip) {
    constexpr int MO = Rx<NB>::MO;
    constexpr int L = NB + 1;
    if (!skip) {
#pragma unroll
        for (int c = 1; c <= NB; ++c)
#pragma unroll
            for (int V = 0; V < MO; ++V) {
                const int a = c + pc(V);
                if (a <= NB && a != 1 && a != L - 1) G[c - 1][V] *= wr[a];
            }
    }
#pragma unroll
    for (int c = 1; c <= NB; ++c)
#pragma unroll
        for (int j = 0; j < NB - 1; ++j)
#pragma unroll
            for (int V = MO - 1; V >= 0; --V)
                if (((V >> j) & 1) && c + pc(V) <= NB) G[c - 1][V] = fma(f[j + 1], G[c - 1][V ^ (1 << j)], G[c - 1][V]);
}

// M += Pi_x s_x with Pi_x = suffix operator of [x0, x) (identity at the chain's first point,
// else R_c[V] = w_c Gr_{l-c-|V|}[V]; l-c-|V| = NB-|R| for c = |U|+1, V = R\U) and
// s_x[U] = o * Bo[U], Bo[U] = B[U << 1] (update k's suffix state at this point, before the
// inverse step).
template <int NB>
__device__ __forceinline__ void rx_M_acc(double (&Mv)[Rx<NB>::MO], const double (&G)[NB][Rx<NB>::MO], const double *wt,
                                         double o, const double (&Bo)[Rx<NB>::MO], bool first) {
    constexpr int MO = Rx<NB>::MO;
    if (first) {
#pragma unroll
        for (int R = 0; R < MO; ++R) Mv[R] = fma(o, Bo[R], Mv[R]);
        return;
    }
    double ow[NB];
#pragma unroll
    for (int a = 1; a <= NB; ++a) ow[a - 1] = o * wt[a];
    double sv[MO];
#pragma unroll
    for (int U = 0; U < MO; ++U) sv[U] = ow[pc(U)] * Bo[U];
#pragma unroll
    for (int R = 0; R < MO; ++R) {
        double acc = Mv[R];
#pragma unroll
        for (int U = 0; U < MO; ++U)
            if ((U & R) == U) acc = fma(G[NB - pc(R) - 1][R ^ U], sv[U], acc);
        Mv[R] = acc;
    }
}

// rx_M_acc on M scaled by 1/w_1 (unscale once at the chain end): the weights of the sources become
// w_{|U|+1} / w_1 = wr[|U|+1], which is 1 for |U|+1 in {1, l-1}.
template <int NB>
__device__ __forceinline__ void rx_M_acc_scaled(double (&Mv)[Rx<NB>::MO], const double (&G)[NB][Rx<NB>::MO],
                                                const double *wr, double w1inv, double o,
                                                const double (&Bo)[Rx<NB>::MO], bool first) {
    constexpr int MO = Rx<NB>::MO;
    constexpr int L = NB + 1;
    if (first) {
        const double o1 = o * w1inv;
#pragma unroll
        for (int R = 0; R < MO; ++R) Mv[R] = fma(o1, Bo[R], Mv[R]);
        return;
    }
    double ow[NB + 1];
#pragma unroll
    for (int a = 1; a <= NB; ++a) ow[a] = (a == 1 || a == L - 1) ? o : o * wr[a];
    double sv[MO];
#pragma unroll
    for (int U = 0; U < MO; ++U) sv[U] = ow[pc(U) + 1] * Bo[U];
#pragma unroll
    for (int R = 0; R < MO; ++R) {
        double acc = Mv[R];
#pragma unroll
        for (int U = 0; U < MO; ++U)
            if ((U & R) == U) acc = fma(G[NB - pc(R) - 1][R ^ U], sv[U], acc);
        Mv[R] = acc;
    }
}

// Chain-end elements: prefix (A'_c[V] = w_c Gr_c[V], offset L) and suffix (A''_c[V] =
// w_c Gr_{l-c-|V|}[V], offset M).
template <int NB>
__device__ __forceinline__ void rx_store(const double (&G)[NB][Rx<NB>::MO], const double (&L)[Rx<NB>::MO],
                                         const double (&Mv)[Rx<NB>::MO], const double *wt, double *ef, double *eb) {
    constexpr int MO = Rx<NB>::MO;
#pragma unroll
    for (int c = 1; c <= NB; ++c)
#pragma unroll
        for (int V = 0; V < MO; ++V) {
            const bool ok = c + pc(V) <= NB;
            ef[(c - 1) * MO + V] = ok ? wt[c] * G[c - 1][V] : 0.0;
            eb[(c - 1) * MO + V] = ok ? wt[c] * G[NB - c - pc(V)][V] : 0.0;
        }
#pragma unroll
    for (int U = 0; U < MO; ++U) {
        ef[NB * MO + U] = L[U];
        eb[NB * MO + U] = Mv[U];
    }
}

// Affine elements: identity, application to a new-part vector, composition (X first, then Y).
template <int NB>
__device__ __forceinline__ void rx_identity(double (&E)[Rx<NB>::SZE]) {
    constexpr int MO = Rx<NB>::MO;
#pragma unroll
    for (int i = 0; i < Rx<NB>::SZE; ++i) E[i] = (i < NB * MO && i % MO == 0) ? 1.0 : 0.0;
}
template <int NB>
__device__ __forceinline__ void rx_apply(const double (&E)[Rx<NB>::SZE], const double (&y)[Rx<NB>::MO],
                                         double (&out)[Rx<NB>::MO]) {
    constexpr int MO = Rx<NB>::MO;
#pragma unroll
    for (int S = 0; S < MO; ++S) {
        double acc = E[NB * MO + S];
#pragma unroll
        for (int U = 0; U < MO; ++U)
            if ((U & S) == U) acc = fma(y[U], E[pc(U) * MO + (S ^ U)], acc);
        out[S] = acc;
    }
}
template <int NB>
__device__ __forceinline__ void rx_compose(const double (&X)[Rx<NB>::SZE], const double (&Y)[Rx<NB>::SZE],
                                           double (&Z)[Rx<NB>::SZE]) {
    constexpr int MO = Rx<NB>::MO;
#pragma unroll
    for (int c = 1; c <= NB; ++c)
#pragma unroll
        for (int V = 0; V < MO; ++V) {
            double acc = 0.0;
            if (c + pc(V) <= NB) {
#pragma unroll
                for (int U = 0; U < MO; ++U)
                    if ((U & V) == U && c + pc(U) <= NB)
                        acc = fma(X[(c - 1) * MO + U], Y[(c + pc(U) - 1) * MO + (V ^ U)], acc);
            }
            Z[(c - 1) * MO + V] = acc;
        }
    double xo[MO], yo[MO];
#pragma unroll
    for (int U = 0; U < MO; ++U) xo[U] = X[NB * MO + U];
    rx_apply<NB>(Y, xo, yo);
#pragma unroll
    for (int U = 0; U < MO; ++U) Z[NB * MO + U] = yo[U];
}

// Sharded contexts with the restricted scan: gathered whole-shard affine elements
// all = [world][2][SZE] (prefix, suffix); new-part carries entering shard `rank`:
//   fin = E_{rank-1} o ... o E_0 (0),   bin = E_{rank+1} o ... o E_{world-1} (0)
// (the new part of e_{} is zero).  Same code on host and device.
template <int NB>
__host__ __device__ inline void compose_rank_affine(const double *all, int world, int rank, double *fin, double *bin) {
    constexpr int MO = Rx<NB>::MO;
    constexpr int SZE = Rx<NB>::SZE;
    double y[MO], z[MO];
    for (int U = 0; U < MO; ++U) y[U] = 0.0;
    for (int r = 0; r < rank; ++r) {
        const double *E = all + ((size_t)r * 2 + 0) * SZE;
        for (int S = 0; S < MO; ++S) {
            double acc = E[NB * MO + S];
            for (int U = 0; U < MO; ++U)
                if ((U & S) == U) acc += y[U] * E[pc(U) * MO + (S ^ U)];
            z[S] = acc;
        }
        for (int U = 0; U < MO; ++U) y[U] = z[U];
    }
    for (int U = 0; U < MO; ++U) fin[U] = y[U];
    for (int U = 0; U < MO; ++U) y[U] = 0.0;
    for (int r = world - 1; r > rank; --r) {
        const double *E = all + ((size_t)r * 2 + 1) * SZE;
        for (int S = 0; S < MO; ++S) {
            double acc = E[NB * MO + S];
            for (int U = 0; U < MO; ++U)
                if ((U & S) == U) acc += y[U] * E[pc(U) * MO + (S ^ U)];
            z[S] = acc;
        }
        for (int U = 0; U < MO; ++U) y[U] = z[U];
    }
    for (int U = 0; U < MO; ++U) bin[U] = y[U];
}

}  // namespace mmot
