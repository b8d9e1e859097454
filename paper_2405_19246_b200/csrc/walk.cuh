// walk.cuh -- device helpers shared by the single-instance kernels (kernels.cu) and the batched
// kernels (batched.cu): weight loads, warp-cooperative slab staging through shared memory,
// the combine of prefix and suffix states, and the Sinkhorn division.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace mmot {

template <int NB, typename T>
__device__ __forceinline__ void load_weights(T (&wt)[NB + 2], const Weights &W) {
#pragma unroll
    for (int a = 0; a <= NB + 1; ++a) load_weight(wt[a], W, a);
}


// ---------------------------------------------------------------------------------------
// Warp-cooperative slab staging.  A warp owns 32 consecutive chains (chunks of P points,
// lane r <-> chain r).  The chains' data are moved through shared memory in slabs of S
// points per chain: each warp-wide cp.async instruction copies 32/S chains' contiguous
// S-point segments (full 32-byte sectors), lanes then read their own chain's values from
// the [32][S+1] tile (odd row pitch: conflict-free 8-byte reads).  Two buffers: the next
// slab is in flight while the current one is consumed.
// ---------------------------------------------------------------------------------------

__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc, bool valid) {
    const unsigned saddr = (unsigned)__cvta_generic_to_shared(sdst);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

// Issue the copies of slab s of NV vectors into buf[NV][32][S+1].  Element e = it*32+lane of
// the [32 chains][S points] slab is chain r = e / S, point j = e % S; chains >= cend (dead
// lanes of the last warp) and points beyond N are zero-filled (src-size 0).
template <int S, int NV>
__device__ __forceinline__ void slab_issue(double *buf, const double *const *vec, int64_t chain0, int64_t P,
                                           int64_t N, int s, int lane) {
    constexpr int RPI = 32 / S;  // chains per warp instruction
    const int r0 = lane / S, j = lane % S;
    const int64_t off = (int64_t)s * S + j;
    const int64_t xb = (chain0 + r0) * P + off;
    const bool offok = off < P;
#pragma unroll
    for (int it = 0; it < S; ++it) {
        const int r = it * RPI + r0;
        const int64_t x = xb + (int64_t)(it * RPI) * P;
        const bool valid = offok && x < N;
#pragma unroll
        for (int v = 0; v < NV; ++v)
            cp_async8(buf + (v * 32 + r) * (S + 1) + j, vec[v] + (valid ? x : 0), valid);
    }
}

// Store an output slab obuf[32][S+1] to global (coalesced, like slab_issue).
template <int S>
__device__ __forceinline__ void slab_store(const double *obuf, double *out, int64_t chain0, int64_t cend, int64_t P,
                                           int64_t N, int s, int lane) {
#pragma unroll
    for (int it = 0; it < S; ++it) {
        const int e = it * 32 + lane;
        const int r = e / S, j = e % S;
        const int64_t off = (int64_t)s * S + j;
        const int64_t x = (chain0 + r) * P + off;
        if (off < P && x < N && chain0 + r < cend) out[x] = obuf[r * (S + 1) + j];
    }
}

template <int NB, int S>
__device__ __forceinline__ void slab_f(double (&f)[NB > 0 ? NB : 1], const double *buf, int lane, int j) {
#pragma unroll
    for (int b = 0; b < NB; ++b) f[b] = buf[(b * 32 + lane) * (S + 1) + j];
}


// Non-uniform grids (paper footnote P:182): the weights of one grid edge with decay lambda =
// exp(-h_e / eta): w_a = lambda^{a(l-a)}, and for duals the cost tangent a(l-a) h_e w_a (the edge's
// share of c(i) = sum_e h_e n(l-n)).
template <int NB, typename T>
__device__ __forceinline__ void pweights_val(T (&w)[NB + 2], double lam, double he) {
    constexpr int L = NB + 1;
    double pw[L * L / 4 + 1];  // lambda^0 .. lambda^{max a(l-a)}
    pw[0] = 1.0;
#pragma unroll
    for (int i = 1; i <= L * L / 4; ++i) pw[i] = pw[i - 1] * lam;
#pragma unroll
    for (int a = 0; a <= NB + 1; ++a) {
        const int ea = a <= L ? a * (L - a) : 0;
        const double wa = a <= L ? pw[ea] : 0.0;
        if constexpr (sizeof(T) == sizeof(double)) {
            reinterpret_cast<double &>(w[a]) = wa;
        } else {
            reinterpret_cast<Dual &>(w[a]) = Dual{wa, (double)ea * he * wa};
        }
    }
}

// mu / J with one Newton step on the reciprocal (relative error ~2^-46) and a residual
// correction of the quotient, which squares that error: q' - mu/J = O(2^-92) + rounding.
__device__ __forceinline__ double div_nr1(double mu, double j) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(j));
    const double e = fma(-j, r, 1.0);
    r = fma(r, e, r);
    const double q = mu * r;
    return fma(r, fma(-j, q, mu), q);
}

// mu / J with one Newton step on the reciprocal only: relative error ~2^-46 (1.4e-14), well inside
// the 1e-10 parity tolerance; two DFMA per point fewer than div_nr1 (FP64-bound update kernels).
__device__ __forceinline__ double div_nr0(double mu, double j) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(j));
    const double e = fma(-j, r, 1.0);
    r = fma(r, e, r);
    return mu * r;
}

// Integer tests on the bit pattern (keep the FP64 pipe free).
__device__ __forceinline__ bool finite_positive(double q) {  // 0 < q < inf
    const unsigned long long b = (unsigned long long)__double_as_longlong(q);
    return b != 0ull && b < 0x7ff0000000000000ull;
}
__device__ __forceinline__ bool nonzero(double q) {
    return ((unsigned long long)__double_as_longlong(q) & 0x7fffffffffffffffull) != 0ull;
}

// Combine J[m] = sum_S F_m[S] H_m[S^c] with two independent accumulators.
template <int NB, typename T>
__device__ __forceinline__ T combine(const T (&F)[1 << NB], const T (&H)[1 << NB]) {
    constexpr int M = 1 << NB;
    T a = zero_of(T{}), b = zero_of(T{});
#pragma unroll
    for (int S = 0; S < M; S += 2) {
        a = mad(F[S], H[(M - 1) ^ S], a);
        if (S + 1 < M) b = mad(F[S + 1], H[(M - 1) ^ (S + 1)], b);
    }
    return T{a} + T{b};
}


// ---------------------------------------------------------------------------------------
// Bulk copies (cp.async.bulk) into shared memory completed through mbarrier transaction counts.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace mmot
