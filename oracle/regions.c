/* O3 -- paper §4.2 region separation with per-region nested first-order recursions.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the
 * CUDA library; plain C99, fp64, single thread.
 *
 * PAPER.md (P:n = line n):
 *   J^{(l)}_{i_l} = sum_{i_1..i_{l-1}} lambda^{sum_{p<q}|i_p-i_q|} prod_{q<l} phi_{q,i_q}
 *   split into l! parts over the order sets D_p
 *   region 1 by the recursion J^{(l)}_{i,1} = lambda^{a} J^{(l)}_{i-1,1} + ... J^{(l-1)}
 *   "similar recursive processes ... for the other J_p"
 *   cost-weighted hat-J by the tangent recursion
 *
 * Reading (A10): a permutation pi lists the marginals in
 * increasing grid position (rank 0 leftmost); ranks r and r+1 may tie iff
 * pi[r] < pi[r+1], otherwise the inequality is strict.  For l = 3 this is
 * exactly D_1..D_6.  Inside a region the exponent is linear in
 * the indices: every grid edge between the positions of ranks r and r+1 is
 * crossed by r+1 indices on its left, contributing e_{r+1} = (r+1)(l-r-1) to
 * sum_{p<q}|i_p - i_q| (the a_p/b_p/c_p table of P:204-214 generalised).  We
 * use the normalised form of Algorithm 2: only relative powers
 * w_a^{gap} with w_a = lambda^{e_a} appear, never absolute powers lambda^{a i}
 * (which overflow at large N).
 *
 * For the free marginal k at rank rho of pi:
 *   prefix chain (ranks 0..rho-1 at positions <= m, ties per strictness):
 *     A_0[x] = phi_{pi[0]}[x];  S_r[x] = w S_r[x-1] + A_r[x];  T_r[x] = w S_r[x-1]
 *     A_{r+1}[x] = phi_{pi[r+1]}[x] * (strict ? T_r[x] : S_r[x]),  Pre = last (no phi_k)
 *   suffix chain: the mirror image from rank l-1 down to rho+1.
 *   J_k[m] += Pre[m] * Suf[m].
 * Tangent (E-weighted) values: each crossed edge adds e to the exponent, so
 *   Shat[x] = w (Shat[x-1] + e S[x-1]) + Ahat[x]  (P:1108-1111 in normalised form).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int next_permutation(int *a, int n) {
    int i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) i--;
    if (i < 0) return 0;
    int j = n - 1;
    while (a[j] <= a[i]) j--;
    int t = a[i]; a[i] = a[j]; a[j] = t;
    for (int p = i + 1, q = n - 1; p < q; p++, q--) { t = a[p]; a[p] = a[q]; a[q] = t; }
    return 1;
}

static double lae(double a, double b) { /* log(e^a + e^b), -inf safe */
    double m = a > b ? a : b;
    if (m == -INFINITY) return -INFINITY;
    return m + log1p(exp(-fabs(a - b)));
}

/* Plain (linear) fp64.
 *   l      number of marginals (2..10)
 *   N      grid points
 *   w      w[a] = lambda^{a(l-a)}, a = 0..l   (caller computes exp(-a(l-a) h/eta) in fp64)
 *   phi    l pointers to N-vectors (phi[k] is not read)
 *   k      free marginal (0-based)
 *   out    N-vector: J_k (overwritten)
 *   out_hat nullable N-vector: hat J_k = sum E(i) lambda^{E(i)} prod phi  (multiply by h for C.K)
 *   region -1 for all l! regions, else only the region with this lexicographic index
 * returns 0 on success, -1 on allocation failure, -2 on bad arguments. */
int mmot_ref_marginal(int l, int64_t N, const double *w, const double *const *phi, int k,
                      double *out, double *out_hat, int region) {
    if (l < 2 || l > 10 || N < 1 || k < 0 || k >= l) return -2;
    const int tan = out_hat != NULL;
    double *A = (double *)malloc(sizeof(double) * (size_t)N);
    double *Suf = (double *)malloc(sizeof(double) * (size_t)N);
    double *Ah = tan ? (double *)malloc(sizeof(double) * (size_t)N) : NULL;
    double *Sufh = tan ? (double *)malloc(sizeof(double) * (size_t)N) : NULL;
    if (!A || !Suf || (tan && (!Ah || !Sufh))) { free(A); free(Suf); free(Ah); free(Sufh); return -1; }
    memset(out, 0, sizeof(double) * (size_t)N);
    if (tan) memset(out_hat, 0, sizeof(double) * (size_t)N);
    int pi[16];
    for (int i = 0; i < l; i++) pi[i] = i;
    int pidx = 0;
    do {
        if (region >= 0 && pidx != region) { pidx++; continue; }
        pidx++;
        int rho = 0;
        while (pi[rho] != k) rho++;
        /* ---- suffix chain: ranks l-1 .. rho+1 -> Suf[x] (rank rho at x) ---- */
        if (rho == l - 1) {
            for (int64_t x = 0; x < N; x++) { Suf[x] = 1.0; if (tan) Sufh[x] = 0.0; }
        } else {
            const double *z0 = phi[pi[l - 1]];
            for (int64_t x = 0; x < N; x++) { Suf[x] = z0[x]; if (tan) Sufh[x] = 0.0; }
            for (int r = l - 1; r >= rho + 1; r--) {
                const double wr = w[r];
                const double er = (double)(r * (l - r));
                const int strict = pi[r - 1] > pi[r];
                const double *nxt = (r - 1 > rho) ? phi[pi[r - 1]] : NULL;
                double s = 0.0, sh = 0.0;
                for (int64_t x = N - 1; x >= 0; x--) {
                    const double cs = wr * s;                 /* sum over y > x */
                    const double csh = tan ? wr * (sh + er * s) : 0.0;
                    s = cs + Suf[x];                           /* sum over y >= x */
                    if (tan) sh = csh + Sufh[x];
                    const double v = strict ? cs : s;
                    const double vh = strict ? csh : sh;
                    Suf[x] = nxt ? nxt[x] * v : v;
                    if (tan) Sufh[x] = nxt ? nxt[x] * vh : vh;
                }
            }
        }
        /* ---- prefix chain: ranks 0 .. rho-1 -> accumulate Pre[x] * Suf[x] ---- */
        if (rho == 0) {
            for (int64_t x = 0; x < N; x++) {
                out[x] += Suf[x];
                if (tan) out_hat[x] += Sufh[x];
            }
        } else {
            const double *a0 = phi[pi[0]];
            for (int64_t x = 0; x < N; x++) { A[x] = a0[x]; if (tan) Ah[x] = 0.0; }
            for (int r = 0; r <= rho - 1; r++) {
                const double wr = w[r + 1];
                const double er = (double)((r + 1) * (l - r - 1));
                const int strict = pi[r] > pi[r + 1];
                const double *nxt = (r + 1 < rho) ? phi[pi[r + 1]] : NULL;
                double s = 0.0, sh = 0.0;
                for (int64_t x = 0; x < N; x++) {
                    const double cs = wr * s;                 /* sum over y < x */
                    const double csh = tan ? wr * (sh + er * s) : 0.0;
                    s = cs + A[x];                             /* sum over y <= x */
                    if (tan) sh = csh + Ah[x];
                    const double v = strict ? cs : s;
                    const double vh = strict ? csh : sh;
                    if (nxt) {
                        A[x] = nxt[x] * v;
                        if (tan) Ah[x] = nxt[x] * vh;
                    } else {
                        out[x] += v * Suf[x];
                        if (tan) out_hat[x] += vh * Suf[x] + v * Sufh[x];
                    }
                }
            }
        }
    } while (next_permutation(pi, l));
    free(A); free(Suf); free(Ah); free(Sufh);
    return 0;
}

/* Log-domain variant: inputs g[q][x] = log phi_q[x] (may be -inf), lw[a] = log w[a]
 * = -a(l-a) h / eta (may be -inf for lambda = 0).  out = log J_k.  Same chains with
 * (+, *) -> (logaddexp, +).  Used where linear fp64 overflows (eta = 1e-3 at C5). */
int mmot_ref_marginal_log(int l, int64_t N, const double *lw, const double *const *g, int k,
                          double *out) {
    if (l < 2 || l > 10 || N < 1 || k < 0 || k >= l) return -2;
    double *A = (double *)malloc(sizeof(double) * (size_t)N);
    double *Suf = (double *)malloc(sizeof(double) * (size_t)N);
    if (!A || !Suf) { free(A); free(Suf); return -1; }
    for (int64_t x = 0; x < N; x++) out[x] = -INFINITY;
    int pi[16];
    for (int i = 0; i < l; i++) pi[i] = i;
    do {
        int rho = 0;
        while (pi[rho] != k) rho++;
        if (rho == l - 1) {
            for (int64_t x = 0; x < N; x++) Suf[x] = 0.0;
        } else {
            const double *z0 = g[pi[l - 1]];
            for (int64_t x = 0; x < N; x++) Suf[x] = z0[x];
            for (int r = l - 1; r >= rho + 1; r--) {
                const double lwr = lw[r];
                const int strict = pi[r - 1] > pi[r];
                const double *nxt = (r - 1 > rho) ? g[pi[r - 1]] : NULL;
                double s = -INFINITY;
                for (int64_t x = N - 1; x >= 0; x--) {
                    const double cs = lwr + s;
                    s = lae(cs, Suf[x]);
                    const double v = strict ? cs : s;
                    Suf[x] = nxt ? nxt[x] + v : v;
                }
            }
        }
        if (rho == 0) {
            for (int64_t x = 0; x < N; x++) out[x] = lae(out[x], Suf[x]);
        } else {
            const double *a0 = g[pi[0]];
            for (int64_t x = 0; x < N; x++) A[x] = a0[x];
            for (int r = 0; r <= rho - 1; r++) {
                const double lwr = lw[r + 1];
                const int strict = pi[r] > pi[r + 1];
                const double *nxt = (r + 1 < rho) ? g[pi[r + 1]] : NULL;
                double s = -INFINITY;
                for (int64_t x = 0; x < N; x++) {
                    const double cs = lwr + s;
                    s = lae(cs, A[x]);
                    const double v = strict ? cs : s;
                    if (nxt) A[x] = nxt[x] + v;
                    else out[x] = lae(out[x], v + Suf[x]);
                }
            }
        }
    } while (next_permutation(pi, l));
    free(A); free(Suf);
    return 0;
}
