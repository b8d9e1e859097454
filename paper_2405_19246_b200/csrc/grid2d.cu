// grid2d.cu -- tensor-vector products on 2-D grids (§4.1), l = 3.
//
// Three distributions on an N x M uniform mesh, flattened column-major (x[i1 + N i2]).
// The kernel factorises, K = K_N(lambda1) (x) K_M(lambda2), so the product with the
// free marginal k is an outer subset recurrence over the M columns whose states are VECTORS over the
// rows, with the paper's inner 1-D product FTVP-1 (K_N x_i x x_j y, lambda1) applied whenever two
// bound marginals meet.  With the bound set {a, b} and outer weights w_s = lambda2^{s(3-s)}:
//   prefix  Fa_x = w1 Fa_{x-1} + a_x,  Fb_x = w1 Fb_{x-1} + b_x                        (vectors over i1)
//           Fab_x = w2 Fab_{x-1} + FTVP(a_x, w1 Fb_{x-1}) + FTVP(Fa_x, b_x)            (vectors over k1)
//   suffix  Ga, Gb, Gab the mirror images (x+1 instead of x-1)
//   combine J_m = w1 Gab_{m+1} + w2 [FTVP(Fa_m, Gb_{m+1}) + FTVP(Ga_{m+1}, Fb_m)] + Fab_m
// i.e. six inner products per column -- Algorithm 6's six FTVP-1 calls per column (P:956-970:
// Fa/Fb/Ga/Gb are its P/Q recursions, Fab/Gab its J_1..J_6 accumulations) in subset form.
//
// Kernels (one launch each):
//   k_g2_scan   thread per row: the four column recursions Fa, Fb, Ga, Gb              (coalesced)
//   k_g2_inner  thread per inner product: the 6M independent 1-D l = 3 products of length N
//               (suffix walk storing its three states, prefix walk + combine)           (batched)
//   k_g2_outer  thread per row: Gab backwards, then Fab + combine + the mode's epilogue
// The cost tangent (Algorithm 3's FTVP-2 inside Algorithm 6; the paper omits the 2-D cost product,
// P:938) is carried as dual numbers d/dlog(lambda1) through the inner products; the lambda2 part is
// the same computation on the transposed mesh (A21).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "internal.h"
#include "walk.cuh"

namespace mmot {

__device__ __forceinline__ void add_s(double &a, double v) { a += v; }
__device__ __forceinline__ void add_s(Dual &a, double v) { a.v += v; }

// column-major N x M -> column-major M x N
__global__ void k_g2_transpose(const double *__restrict__ in, double *__restrict__ out, int64_t N, int64_t M) {
    __shared__ double tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t r = r0 + threadIdx.x, c = c0 + j;
        tile[j][threadIdx.x] = (r < N && c < M) ? in[r + N * c] : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t c = c0 + threadIdx.x, r = r0 + j;  // out[c + M r]
        if (r < N && c < M) out[c + M * r] = tile[threadIdx.x][j];
    }
}

cudaError_t launch_g2_transpose(const double *in, double *out, int64_t N, int64_t M, cudaStream_t s,
                                int64_t *launches) {
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
    k_g2_transpose<<<grid, dim3(32, 8), 0, s>>>(in, out, N, M);
    ++*launches;
    return cudaGetLastError();
}

__global__ void k_g2_scan(G2Plan p) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.N || *p.stop) return;
    const int64_t N = p.N, M = p.M;
    double fa = 0.0, fb = 0.0;
    for (int64_t x = 0; x < M; ++x) {
        fa = fma(p.wo1, fa, p.a[r + N * x]);
        fb = fma(p.wo1, fb, p.b[r + N * x]);
        p.Fa[r + N * x] = fa;
        p.Fb[r + N * x] = fb;
    }
    double ga = 0.0, gb = 0.0;
    for (int64_t x = M - 1; x >= 0; --x) {
        ga = fma(p.wo1, ga, p.a[r + N * x]);
        gb = fma(p.wo1, gb, p.b[r + N * x]);
        p.Ga[r + N * x] = ga;
        p.Gb[r + N * x] = gb;
    }
}

// One 1-D l = 3 product J[m] = sum_{i,j} lambda1^{|i-j|+|i-m|+|j-m|} X[i] Y[j] (FTVP-1) by
// the two-state-set recurrence: suffix states (B_X, B_Y, B_XY) stored per point, then the prefix
// walk and the combine J = w1 B_XY + w2 (F_X B_Y + F_Y B_X) + F_XY.
template <typename T>
__global__ void k_g2_inner(G2Plan p) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = p.N, M = p.M;
    if (idx >= 6 * M || *p.stop) return;
    const int kind = (int)(idx / M);
    const int64_t x = idx % M;
    const double *X = nullptr, *Y = nullptr;
    double sy = 1.0;
    switch (kind) {
        case 0: X = p.a + N * x; Y = x > 0 ? p.Fb + N * (x - 1) : nullptr; sy = p.wo1; break;      // prefix, a at x
        case 1: X = p.Fa + N * x; Y = p.b + N * x; break;                                            // prefix, b at x
        case 2: X = p.a + N * x; Y = x + 1 < M ? p.Gb + N * (x + 1) : nullptr; sy = p.wo1; break;  // suffix, a at x
        case 3: X = p.Ga + N * x; Y = p.b + N * x; break;                                            // suffix, b at x
        case 4: X = p.Fa + N * x; Y = x + 1 < M ? p.Gb + N * (x + 1) : nullptr; break;              // combine S = {a}
        default: X = x + 1 < M ? p.Ga + N * (x + 1) : nullptr; Y = p.Fb + N * x; break;            // combine S = {b}
    }
    T *out = static_cast<T *>(p.Y) + (kind * M + x) * N;
    if (!X || !Y) {
        for (int64_t m = 0; m < N; ++m) out[m] = zero_of(T{});
        return;
    }
    T w1, w2;
    load_weight(w1, p.Wi, 1);
    load_weight(w2, p.Wi, 2);
    T *st = static_cast<T *>(p.st) + idx * N * 3;
    T bx = zero_of(T{}), by = zero_of(T{}), bxy = zero_of(T{});
    for (int64_t m = N - 1; m >= 0; --m) {
        st[3 * m + 0] = bx;  // B_{m+1}
        st[3 * m + 1] = by;
        st[3 * m + 2] = bxy;
        const double xv = X[m], yv = sy * Y[m];
        bx = mul(w1, bx);
        by = mul(w1, by);
        bxy = mul(w2, bxy);
        bxy = mads(xv, by, bxy);  // place X: B_XY += x B_Y
        add_s(bx, xv);             // B_X += x (times B_empty = 1)
        bxy = mads(yv, bx, bxy);  // place Y: B_XY += y B_X
        add_s(by, yv);
    }
    T fx = zero_of(T{}), fy = zero_of(T{}), fxy = zero_of(T{});
    for (int64_t m = 0; m < N; ++m) {
        const double xv = X[m], yv = sy * Y[m];
        fx = mul(w1, fx);
        fy = mul(w1, fy);
        fxy = mul(w2, fxy);
        fxy = mads(xv, fy, fxy);
        add_s(fx, xv);
        fxy = mads(yv, fx, fxy);
        add_s(fy, yv);
        const T b0 = st[3 * m + 0], b1 = st[3 * m + 1], b2 = st[3 * m + 2];
        T J = mul(w1, b2);
        J = mad(w2, mad(fx, b1, mul(fy, b0)), J);
        out[m] = J + fxy;
    }
}

// Outer recurrences of the output-space states and the combine, thread per row r; epilogue per mode.
template <typename T>
__global__ void k_g2_outer(G2Plan p, int mode) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = p.N, M = p.M;
    if (r >= N || *p.stop) return;
    const T *Yv = static_cast<const T *>(p.Y);
    T *gab = static_cast<T *>(p.Gab);
    T g = zero_of(T{});
    gab[N * M + r] = g;  // G_M = 0
    for (int64_t x = M - 1; x >= 0; --x) {
        g = mads(p.wo2, g, Yv[(2 * M + x) * N + r] + Yv[(3 * M + x) * N + r]);
        gab[N * x + r] = g;
    }
    T f = zero_of(T{});
    double acc = 0.0;
    bool bad = false;
    for (int64_t x = 0; x < M; ++x) {
        f = mads(p.wo2, f, Yv[(0 * M + x) * N + r] + Yv[(1 * M + x) * N + r]);
        T J = mads(p.wo1, gab[N * (x + 1) + r], f);
        J = mads(p.wo2, Yv[(4 * M + x) * N + r] + Yv[(5 * M + x) * N + r], J);
        const double jv = value_of(J);
        const int64_t i = r + N * x;
        if (mode == MODE_UPD) {
            const double mu = p.muk[i];
            const double q = div_nr1(mu, jv);
            const bool nz = nonzero(mu);
            bad |= nz && !finite_positive(q);
            p.outk[i] = nz ? q : 0.0;
        } else if (mode == MODE_MARG) {
            const double ph = p.phik[i];
            bad |= ph > 0.0 && !finite_positive(jv);
            p.outk[i] = ph * jv;
        } else if (mode == MODE_RES) {
            acc += fabs(p.phik[i] * jv - p.muk[i]);
        } else {
            if constexpr (sizeof(T) == sizeof(Dual)) acc += p.phik[i] * reinterpret_cast<const Dual &>(J).d;
        }
    }
    if (mode == MODE_RES || mode == MODE_COST) p.partial[r] = acc;
    if (bad) {
        if (atomicCAS(p.status, 0, 6) == 0) *p.fail_iter = p.iter;
        *(volatile int *)p.stop = 1;
    }
}

cudaError_t launch_g2_product(const G2Plan &p, int mode, cudaStream_t s, int64_t *launches) {
    const unsigned rb = (unsigned)((p.N + 127) / 128);
    k_g2_scan<<<rb, 128, 0, s>>>(p);
    const unsigned ib = (unsigned)((6 * p.M + 63) / 64);
    if (mode == MODE_COST) {
        k_g2_inner<Dual><<<ib, 64, 0, s>>>(p);
        k_g2_outer<Dual><<<rb, 128, 0, s>>>(p, mode);
    } else {
        k_g2_inner<double><<<ib, 64, 0, s>>>(p);
        k_g2_outer<double><<<rb, 128, 0, s>>>(p, mode);
    }
    *launches += 3;
    return cudaGetLastError();
}

}  // namespace mmot
