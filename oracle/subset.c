/* O4 -- subset-lattice dynamic programme for the l-marginal tensor-vector product (SURVEY §0.1,
 * §8(c) O4).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA library;
 * plain C99, fp64, single thread per call (callers may run independent calls on several threads).
 *
 * What it computes (PAPER.md, P:n = line n):
 *   J_k[m] = sum_{i : i_k = m} lambda^{E(i)} prod_{q != k} phi_q[i_q],
 *   E(i) = sum_{p<q} |i_p - i_q|
 * through the edge form of the exponent (pinned by tests/test_oracle_regions.py):
 *   E(i) = sum_{x=0}^{N-2} a_x (l - a_x),  a_x = #{p : i_p <= x},
 * so crossing the grid edge (x, x+1) with a indices on its left multiplies by w_a = lambda^{a(l-a)}.
 * Sweeping the grid, the state is the set S of bound marginals (B = {0..l-1} \ {k}) already
 * placed; with the states written out as the plain subset sums
 *   F_x[S] = sum_{T subset S} w_{|S\T|} F_{x-1}[S\T] prod_{q in T} phi_q[x],   F_{-1} = e_empty
 *   G_x[R] = sum_{T subset R} w_{|R\T|} G_{x+1}[R\T] prod_{q in T} phi_q[x],   G_N    = e_empty
 *   J_k[m] = sum_{S subset B} F_m[S] w_{|S|+1} G_{m+1}[B\S]
 * (the free index m sits between the prefix and the suffix: the edge (m, m+1) is crossed by the
 * |S| + 1 indices at or left of m).  All terms are positive: the DP re-associates the same sum.
 * The tangent Jhat = sum_i E(i) lambda^{E(i)} prod phi = lambda dJ/dlambda is carried
 * as dual numbers (value, d/dlog lambda) with dw_a = e_a w_a, e_a = a(l-a).
 * The log variant takes g_q = log phi_q and log-weights lw_a = log w_a and evaluates the same
 * sums with log-sum-exp (Remark 1's purpose, as a pure log domain).
 *
 * Cost: 3^(l-1) terms per point and direction; memory: the suffix states G, (N+1) 2^(l-1) doubles.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXL 8

typedef struct { double v, d; } dual;

static int popc(unsigned x) { int c = 0; while (x) { c += (int)(x & 1u); x >>= 1; } return c; }

/* bound marginals of the product J_k, increasing index */
static int bound_list(int l, int k, int *b) {
    int n = 0;
    for (int q = 0; q < l; ++q) if (q != k) b[n++] = q;
    return n;
}

/* prod_{q in T} phi_{b[q]}[x] for every subset T of the n bound marginals */
static void subset_products(int n, const int *b, const double *const *phi, int64_t x, double *pt) {
    const unsigned M = 1u << n;
    pt[0] = 1.0;
    for (unsigned T = 1; T < M; ++T) {
        int q = 0;
        while (!(T & (1u << q))) ++q;                 /* lowest element of T */
        pt[T] = pt[T & ~(1u << q)] * phi[b[q]][x];
    }
}

/* one DP step: out[S] = sum_{T subset S} w_{|S\T|} in[S\T] pt[T] */
static void step_plain(int n, const double *w, const double *in, const double *pt, double *out) {
    const unsigned M = 1u << n;
    for (unsigned S = 0; S < M; ++S) {
        double acc = 0.0;
        for (unsigned T = S;; T = (T - 1) & S) {       /* all subsets T of S */
            const unsigned R = S & ~T;
            acc += w[popc(R)] * in[R] * pt[T];
            if (T == 0) break;
        }
        out[S] = acc;
    }
}

static void step_dual(int n, const dual *w, const dual *in, const double *pt, dual *out) {
    const unsigned M = 1u << n;
    for (unsigned S = 0; S < M; ++S) {
        dual acc = {0.0, 0.0};
        for (unsigned T = S;; T = (T - 1) & S) {
            const unsigned R = S & ~T;
            const dual a = w[popc(R)], x = in[R];
            acc.v += a.v * x.v * pt[T];
            acc.d += (a.d * x.v + a.v * x.d) * pt[T];
            if (T == 0) break;
        }
        out[S] = acc;
    }
}

/* Plain fp64 (and, if outhat != NULL, the tangent Jhat).
 *   w[a] = lambda^{a(l-a)}, a = 0..l;  phi: l pointers to N-vectors (phi[k] unread);  out: N.
 * Returns 0, or -1 on a bad argument / allocation failure. */
int mmot_ref_subset(int l, int64_t N, const double *w, const double *const *phi, int k, double *out,
                    double *outhat) {
    if (l < 2 || l > MAXL || N < 1 || k < 0 || k >= l || !w || !phi || !out) return -1;
    int b[MAXL];
    const int n = bound_list(l, k, b);
    const unsigned M = 1u << n;
    double pt[1u << (MAXL - 1)];
    dual wd[MAXL + 1];
    for (int a = 0; a <= l; ++a) { wd[a].v = w[a]; wd[a].d = (double)(a * (l - a)) * w[a]; }
    const int dual_mode = outhat != NULL;
    const size_t esz = dual_mode ? sizeof(dual) : sizeof(double);
    char *G = (char *)malloc((size_t)(N + 1) * M * esz);   /* suffix states G_x, x = 0..N */
    char *Fa = (char *)malloc(2 * (size_t)M * esz);
    if (!G || !Fa) { free(G); free(Fa); return -1; }
    memset(G + (size_t)N * M * esz, 0, M * esz);
    if (dual_mode) ((dual *)(G + (size_t)N * M * esz))[0].v = 1.0;
    else ((double *)(G + (size_t)N * M * esz))[0] = 1.0;
    for (int64_t x = N - 1; x >= 0; --x) {
        subset_products(n, b, phi, x, pt);
        if (dual_mode) step_dual(n, wd, (const dual *)(G + (size_t)(x + 1) * M * esz), pt, (dual *)(G + (size_t)x * M * esz));
        else step_plain(n, w, (const double *)(G + (size_t)(x + 1) * M * esz), pt, (double *)(G + (size_t)x * M * esz));
    }
    char *Fp = Fa, *Fc = Fa + M * esz;                     /* F_{x-1}, F_x */
    memset(Fp, 0, M * esz);
    if (dual_mode) ((dual *)Fp)[0].v = 1.0;
    else ((double *)Fp)[0] = 1.0;
    const unsigned full = M - 1;
    for (int64_t m = 0; m < N; ++m) {
        subset_products(n, b, phi, m, pt);
        if (dual_mode) {
            step_dual(n, wd, (const dual *)Fp, pt, (dual *)Fc);
            const dual *F = (const dual *)Fc, *Gn = (const dual *)(G + (size_t)(m + 1) * M * esz);
            double jv = 0.0, jd = 0.0;
            for (unsigned S = 0; S < M; ++S) {
                const dual a = wd[popc(S) + 1], f = F[S], g = Gn[full & ~S];
                jv += f.v * a.v * g.v;
                jd += f.d * a.v * g.v + f.v * a.d * g.v + f.v * a.v * g.d;
            }
            out[m] = jv;
            outhat[m] = jd;
        } else {
            step_plain(n, w, (const double *)Fp, pt, (double *)Fc);
            const double *F = (const double *)Fc, *Gn = (const double *)(G + (size_t)(m + 1) * M * esz);
            double j = 0.0;
            for (unsigned S = 0; S < M; ++S) j += F[S] * w[popc(S) + 1] * Gn[full & ~S];
            out[m] = j;
        }
        char *t = Fp; Fp = Fc; Fc = t;
    }
    free(G);
    free(Fa);
    return 0;
}

static double lae(double a, double b) { /* log(e^a + e^b), -inf safe */
    const double m = a > b ? a : b;
    if (m == -INFINITY) return -INFINITY;
    return m + log1p(exp(-fabs(a - b)));
}

static void step_log(int n, const double *lw, const double *in, const double *lpt, double *out) {
    const unsigned M = 1u << n;
    for (unsigned S = 0; S < M; ++S) {
        double acc = -INFINITY;
        for (unsigned T = S;; T = (T - 1) & S) {
            const unsigned R = S & ~T;
            acc = lae(acc, lw[popc(R)] + in[R] + lpt[T]);
            if (T == 0) break;
        }
        out[S] = acc;
    }
}

/* Log domain: g = l pointers to log phi (-inf allowed), lw[a] = log w_a; out = log J_k. */
int mmot_ref_subset_log(int l, int64_t N, const double *lw, const double *const *g, int k, double *out) {
    if (l < 2 || l > MAXL || N < 1 || k < 0 || k >= l || !lw || !g || !out) return -1;
    int b[MAXL];
    const int n = bound_list(l, k, b);
    const unsigned M = 1u << n;
    double lpt[1u << (MAXL - 1)];
    double *G = (double *)malloc((size_t)(N + 1) * M * sizeof(double));
    double *Fa = (double *)malloc(2 * (size_t)M * sizeof(double));
    if (!G || !Fa) { free(G); free(Fa); return -1; }
    for (unsigned S = 0; S < M; ++S) G[(size_t)N * M + S] = S == 0 ? 0.0 : -INFINITY;
    for (int64_t x = N - 1; x >= 0; --x) {
        lpt[0] = 0.0;
        for (unsigned T = 1; T < M; ++T) {
            int q = 0;
            while (!(T & (1u << q))) ++q;
            lpt[T] = lpt[T & ~(1u << q)] + g[b[q]][x];
        }
        step_log(n, lw, G + (size_t)(x + 1) * M, lpt, G + (size_t)x * M);
    }
    double *Fp = Fa, *Fc = Fa + M;
    for (unsigned S = 0; S < M; ++S) Fp[S] = S == 0 ? 0.0 : -INFINITY;
    const unsigned full = M - 1;
    for (int64_t m = 0; m < N; ++m) {
        lpt[0] = 0.0;
        for (unsigned T = 1; T < M; ++T) {
            int q = 0;
            while (!(T & (1u << q))) ++q;
            lpt[T] = lpt[T & ~(1u << q)] + g[b[q]][m];
        }
        step_log(n, lw, Fp, lpt, Fc);
        double j = -INFINITY;
        for (unsigned S = 0; S < M; ++S) j = lae(j, Fc[S] + lw[popc(S) + 1] + G[(size_t)(m + 1) * M + (full & ~S)]);
        out[m] = j;
        double *t = Fp; Fp = Fc; Fc = t;
    }
    free(G);
    free(Fa);
    return 0;
}
