// pair.cu -- the pair family: large batches of small instances (BASELINE C5: 8192 x (l = 5,
// N = 4096), per-instance eta), TWO threads per instance and no chain operators.
//
// The persistent batched kernel (batched.cu) cuts an instance into 32 chains, one per lane, and
// joins them through chain operators: the operator walk costs ~160 fp64 instructions per point at
// l = 5 against ~50 for a state walk, and the 31-step carry propagation is serial.  With two chains
// per instance no operator is needed, because each half has one end whose carry is the empty-set
// state e_{} (Algorithm 1's products in subset form):
//     phase 1   left thread  (half A = points 0 .. H-1):  prefix walk from e_{}  -> F_{H-1}
//               right thread (half B = points H .. N-1):  suffix walk from e_{}  -> B_H
//               (both store their own walk's state every kPS points: checkpoints)
//     exchange  F_{H-1} and B_H swap threads (one shuffle per state)
//     phase 2   left:  suffix walk from B_H down to 0, prefix states rebuilt from the checkpoints
//               right: prefix walk from F_{H-1} up to N-1, suffix states rebuilt likewise
//               combine J_k[x] = sum_S Own_x[S] (D Other)[S^c] and phi_k = mu_k / J_k
// The right half is stored MIRRORED (position p <-> point N-1-p), so in position space both threads
// run the same code: a suffix recursion B_x = place_x(D B_{x+1}) is a prefix recursion over the
// mirrored points, and the combine weight w_{|S|+1} = w_{l-1-|S|} is symmetric (w_a = w_{l-a}).
//
// Range (a8).  At eta = 1e-3 |log phi| reaches ~1.8e3 and phi changes by up to 2^1.4 per point, so
// a half (2048 points) spans far more than fp64's range.  Every scaling is stored as
//     phi_q[x] = m_q[x] * 2^{E_q[slab]}     (mantissa field + one exponent per kPS = 8 positions)
// and a state is kept relative to 2^{sum_{q in S} E_q[slab]} of the slab it is in; crossing a slab
// boundary multiplies F[S] by the exact power of two 2^{sum_{q in S} (E_q[old] - E_q[new])}
// (batched.cu's chain-boundary conversion, here every 8 points).  The update writes phi_k's
// mantissas normalised per slab (max mantissa in [1, 2)).
//
// Layout (this family's own, converted at the API boundary): vector q of block blk (16 instances)
// is [position p][lane] with lane = 2 i + half, so a warp's load of one position is 32 consecutive
// elements (fully coalesced), and each lane walks its own half.  Checkpoints [slab][S][lane].
// Data are staged through shared memory by bulk copies (one per tile, mbarrier completion), one
// slab ahead.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <climits>

#include "internal.h"
#include "walk.cuh"

namespace mmot {

constexpr int kPS = 8;      // slab: positions per exponent block and checkpoint
constexpr int kPQ = 4;      // rebuild sub-block (keeps kPQ own states in registers)
constexpr int kPWarps = 2;  // warps per CTA
constexpr int kPStages = 2; // shared-memory stages per warp (one slab in flight)

// exact 2^n, n clamped to the normal range
__device__ __forceinline__ double pr_pow2c(int n) {
    n = max(-1022, min(1023, n));
    return __longlong_as_double((long long)(n + 1023) << 52);
}
__device__ __forceinline__ float pr_pow2cf(int n) {
    n = max(-126, min(127, n));
    return __int_as_float((n + 127) << 23);
}
// floor(log2 x) of a positive normal value; INT_MIN for 0 / denormals
__device__ __forceinline__ int pr_ilog2(double x) {
    const int e = (int)((__double_as_longlong(x) >> 52) & 0x7ff);
    return e == 0 ? INT_MIN : e - 1023;
}
__device__ __forceinline__ int pr_ilog2(float x) {
    const int e = (__float_as_int(x) >> 23) & 0xff;
    return e == 0 ? INT_MIN : e - 127;
}

// Compute-type traits of the walks: CT = double (fp64 arithmetic) or float (fp32 arithmetic on
// MMOT_F32 contexts: states are kept relative to the slab exponents, so their range stays a few tens
// of bits -- measured [-14, +36] bits on C5 instances over eta in [1e-3, 1e-2] -- far inside fp32's).
template <typename CT>
struct PrT;
template <>
struct PrT<double> {
    static constexpr int kMaxShift = 255;  // per marginal: the subset products stay normal
    static __device__ __forceinline__ double pow2(int n) { return pr_pow2c(n); }
    static __device__ __forceinline__ double exact2(int n) { return __longlong_as_double((long long)(n + 1023) << 52); }
    static __device__ __forceinline__ bool finite_pos(double q) { return finite_positive(q); }
    static __device__ __forceinline__ bool nz(double q) { return nonzero(q); }
    // mu / J~ (phi_k relative to 2^{-sum E_b}) in fp64 for both compute types: the quotient's own
    // range (the product of the bound scalings' relative values) can leave fp32 even when J~ fits
    static __device__ __forceinline__ double div(double mu, double j) { return div_nr1(mu, j); }
};
template <>
struct PrT<float> {
    static constexpr int kMaxShift = 31;
    static __device__ __forceinline__ float pow2(int n) { return pr_pow2cf(n); }
    static __device__ __forceinline__ float exact2(int n) { return __int_as_float((n + 127) << 23); }
    static __device__ __forceinline__ bool finite_pos(float q) {
        const unsigned b = (unsigned)__float_as_int(q);
        return b != 0u && b < 0x7f800000u;
    }
    static __device__ __forceinline__ bool nz(float q) { return ((unsigned)__float_as_int(q) & 0x7fffffffu) != 0u; }
    // mu / J~ in fp64 (one Newton step on the reciprocal, 2^-46: far inside the fp32 tolerance)
    static __device__ __forceinline__ double div(float mu, float j) { return div_nr0((double)mu, (double)j); }
};

// One grid point of the subset recurrence (dp.cuh dp_diag / dp_place) in the compute type:
// diag st[S] *= w_{|S|} (w_0 = 1: the empty set is skipped), place st[S] += f_b st[S \ b].
template <int NB, typename CT>
__device__ __forceinline__ void pr_step(CT (&st)[1 << NB], const CT (&wt)[NB + 2], const CT (&f)[NB]) {
#pragma unroll
    for (int S = 1; S < (1 << NB); ++S) st[S] = wt[pc(S)] * st[S];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
        for (int S = (1 << NB) - 1; S >= 0; --S)
            if ((S >> b) & 1) st[S] = fma(f[b], st[S ^ (1 << b)], st[S]);
    }
}
template <int NB, typename CT>
__device__ __forceinline__ void pr_place(CT (&st)[1 << NB], const CT (&f)[NB]) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
        for (int S = (1 << NB) - 1; S >= 0; --S)
            if ((S >> b) & 1) st[S] = fma(f[b], st[S ^ (1 << b)], st[S]);
    }
}
// J = sum_S F[S] H[S^c], two independent accumulators (walk.cuh combine)
template <int NB, typename CT>
__device__ __forceinline__ CT pr_combine(const CT (&F)[1 << NB], const CT (&H)[1 << NB]) {
    constexpr int M = 1 << NB;
    CT a = CT(0), b = CT(0);
#pragma unroll
    for (int S = 0; S < M; S += 2) {
        a = fma(F[S], H[(M - 1) ^ S], a);
        if (S + 1 < M) b = fma(F[S + 1], H[(M - 1) ^ (S + 1)], b);
    }
    return a + b;
}

// st[S] *= 2^{sum_{b in S} d[b]}.  Neighbouring slabs' exponents differ by a few bits, so the
// usual path forms 2^{d_b} once and the 2^NB subset factors by products (exact: every partial sum
// stays inside the normal range); larger jumps take two clamped factors per state.
template <int NB, typename CT>
__device__ __forceinline__ void pr_shift(CT (&st)[1 << NB], const int (&d)[NB]) {
    constexpr int M = 1 << NB;
    constexpr int LIM = PrT<CT>::kMaxShift;
    bool small = true;
#pragma unroll
    for (int b = 0; b < NB; ++b) small &= d[b] >= -LIM && d[b] <= LIM;
    if (small) {
        CT fb[NB], fac[M];
#pragma unroll
        for (int b = 0; b < NB; ++b) fb[b] = PrT<CT>::exact2(d[b]);
#pragma unroll
        for (int S = 1; S < M; ++S) {
            const int low = S & -S;
            const int b = low == 1 ? 0 : low == 2 ? 1 : low == 4 ? 2 : low == 8 ? 3 : 4;
            fac[S] = S == low ? fb[b] : fac[S ^ low] * fb[b];
            st[S] *= fac[S];
        }
        return;
    }
#pragma unroll
    for (int S = 1; S < M; ++S) {
        int n = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
            if ((S >> b) & 1) n += d[b];
        const int h1 = n >> 1;
        st[S] = (st[S] * PrT<CT>::pow2(h1)) * PrT<CT>::pow2(n - h1);
    }
}

// Shared-memory stage of one slab: bound mantissas [NB][kPS][32] (PT), mu [kPS][32] (MT),
// checkpoint [M][32] (double) -- each tile one contiguous range of global memory.
template <int NB, typename PT, typename MT, typename CT>
struct PStage {
    static constexpr int M = 1 << NB;
    static constexpr int TILE_P = kPS * 32 * (int)sizeof(PT);  // one vector's slab: contiguous in global
    static constexpr int TILE_M = kPS * 32 * (int)sizeof(MT);
    static constexpr int TILE_C = M * 32 * (int)sizeof(CT);     // the slab's checkpoint
    static constexpr int OFF_MU = NB * TILE_P;
    static constexpr int OFF_CK = OFF_MU + TILE_M;
    // the slab's exponent record of all l marginals: [q][E, G][lane] ints (one contiguous tile)
    static constexpr int TILE_X = (NB + 1) * 2 * 32 * (int)sizeof(int);
    static constexpr int OFF_X = OFF_CK + TILE_C;
    static constexpr int BYTES = OFF_X + TILE_X;
};

template <int NB, typename PT, typename MT, typename CT>
size_t pair_smem() {
    return (size_t)kPWarps * kPStages * PStage<NB, PT, MT, CT>::BYTES;
}

// State-scale exponents of the fp32 walks.  With E[j] the slab exponents of one
// scaling over the whole line (this lane's half, slabs 0 = open end .. n-1 = middle, and the partner
// lane's half mirrored beyond the middle), G[j] = ceil(max_j' (E[j'] - c8 |j - j'|)), c8 = the kernel's
// decay over one slab in bits, 8 (l-1) h / (eta ln 2): G never falls faster than the kernel decays, so
// a state relative to 2^{G} cannot grow from far-away mass (a marginal's deep tail, where E falls
// faster), and m 2^{E - G} only drops values that far-away mass dominates.  Two lanes (the pair) call
// this together: one shuffle exchanges the envelope at the middle.
// Exponent records: E (mantissa exponents) and G (state scales of the fp32 walks) of marginal q,
// block blk, slab j live at pp.E[((blk * nslab + j) * l + q) * 64 + {0: E, 32: G} + lane], so the
// records of all l marginals of one slab are one contiguous tile (one bulk copy per slab).
__device__ __forceinline__ int64_t pr_xrec(const PairPlan &pp, int q, int64_t blk, int64_t j) {
    return ((blk * pp.nslab + j) * pp.l + q) * 64;
}

// e, g: this lane's E and G of one marginal, slab stride `st` ints.
__device__ __forceinline__ void pair_envelope(const int *__restrict__ e, int *__restrict__ g, int n, double c8,
                                              int64_t st) {
    // loads in groups of kEG (independent, in flight together), the cone serially over each group
#ifndef MMOT_PAIR_EG
#define MMOT_PAIR_EG 32
#endif
    constexpr int kEG = MMOT_PAIR_EG;
    double a = -1e300;
    for (int j0 = 0; j0 < n; j0 += kEG) {                              // open end -> middle
        int v[kEG];
#pragma unroll
        for (int i = 0; i < kEG; ++i) v[i] = j0 + i < n ? __ldcg(e + (j0 + i) * st) : INT_MIN;
#pragma unroll
        for (int i = 0; i < kEG; ++i)
            if (j0 + i < n) {
                a = fmax((double)v[i], a - c8);
                g[(j0 + i) * st] = (int)ceil(a);
            }
    }
    a = __shfl_xor_sync(0xffffffffu, a, 1);                           // the partner's, at its middle
    for (int j1 = n - 1; j1 >= 0; j1 -= kEG) {                         // middle (and beyond) -> open end
        int v[kEG], w[kEG];
#pragma unroll
        for (int i = 0; i < kEG; ++i) {
            v[i] = j1 - i >= 0 ? __ldcg(e + (j1 - i) * st) : INT_MIN;
            w[i] = j1 - i >= 0 ? __ldcg(g + (j1 - i) * st) : INT_MIN;
        }
#pragma unroll
        for (int i = 0; i < kEG; ++i)
            if (j1 - i >= 0) {
                a = fmax((double)v[i], a - c8);
                g[(j1 - i) * st] = max(w[i], (int)ceil(a));
            }
    }
}

// One Gauss-Seidel update phi_k <- mu_k / J_k of the warp's 16 instances.
template <int NB, typename PT, typename MT, typename CT>
__device__ __forceinline__ bool pair_update(const PairPlan &pp, int64_t blk, int k, const CT (&wt)[NB + 2],
                                            char *stg, uint64_t *bar, unsigned &par, CT *ck, int lane, bool dead,
                                            double c8) {
    using ST = PStage<NB, PT, MT, CT>;
    using TR = PrT<CT>;
    // ENV (fp32 arithmetic): the states are kept relative to 2^{sum_b G_b[slab]}, G = the decay
    // envelope of the slab exponents (pair_envelope), and the mantissas enter the walks as
    // m 2^{E - G} <= m; fp64 arithmetic keeps G = E.
    constexpr bool ENV = sizeof(CT) == sizeof(float);
    constexpr int L = NB + 1, M = 1 << NB;
    const int nslab = pp.nslab;
    const int64_t npos = (int64_t)nslab * kPS;
    const PT *phit = static_cast<const PT *>(pp.phit);
    // global bases of the bound vectors' tiles (mantissas [position][lane], exponents [slab][lane])
    const PT *vbase[NB];
    int qb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        qb[b] = (k + 1 + b) % L;
        vbase[b] = phit + ((int64_t)qb[b] * pp.nblk + blk) * npos * 32;
    }
    const int *xbase = pp.E + pr_xrec(pp, 0, blk, 0);  // slab j's record tile at + j * l * 64
    // f multiplier of a slab: 2^{E - G} (exact; below 2^-126 the mantissas are dropped)
    auto fscale = [&](int e, int g) -> CT {
        if constexpr (ENV) return e - g >= -126 ? __int_as_float((e - g + 127) << 23) : 0.0f;
        else return CT(1);
    };
    // one slab into stage `slot`: bulk copies issued by lane 0, completion on the slot's mbarrier
    // (every tile is contiguous in global memory: [position][lane], [state][lane], [lane])
    auto issue = [&](int j, int slot, bool p2) {
        if (lane == 0) {
            char *sb = stg + slot * ST::BYTES;
            mbar_arrive_expect_tx(&bar[slot], (uint32_t)(NB * ST::TILE_P + ST::TILE_X + (p2 ? ST::TILE_M + ST::TILE_C : 0)));
#pragma unroll
            for (int b = 0; b < NB; ++b)
                bulk_g2s(sb + b * ST::TILE_P, vbase[b] + (int64_t)j * kPS * 32, ST::TILE_P, &bar[slot]);
            bulk_g2s(sb + ST::OFF_X, xbase + (int64_t)j * L * 64, ST::TILE_X, &bar[slot]);
            if (p2) {
                const MT *vm = static_cast<const MT *>(pp.mu) + ((int64_t)k * pp.nblk + blk) * npos * 32;
                bulk_g2s(sb + ST::OFF_MU, vm + (int64_t)j * kPS * 32, ST::TILE_M, &bar[slot]);
                bulk_g2s(sb + ST::OFF_CK, ck + (int64_t)j * M * 32, ST::TILE_C, &bar[slot]);
            }
        }
    };
    // par carries each stage's mbarrier phase across updates
    auto wait = [&](int slot) -> const char * {
        mbar_wait(&bar[slot], (par >> slot) & 1u);
        par ^= 1u << slot;
        return stg + slot * ST::BYTES;
    };
    // the slab's state scales (ecur) and mantissa multipliers (fsc) from a stage
    int ecur[NB];
    CT fsc[NB];
    auto slab_scales = [&](const char *sb, int (&e)[NB], CT (&f)[NB]) {
        const int *sx = reinterpret_cast<const int *>(sb + ST::OFF_X);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int x = sx[qb[b] * 64 + lane];
            e[b] = ENV ? sx[qb[b] * 64 + 32 + lane] : x;
            f[b] = fscale(x, e[b]);
        }
    };
    // ---- phase 1: own walk over positions 0 .. npos-1, checkpoint before every slab
    CT st[M];
#pragma unroll
    for (int S = 0; S < M; ++S) st[S] = S == 0 ? CT(1) : CT(0);
    issue(0, 0, false);
#pragma unroll 1
    for (int j = 0; j < nslab; ++j) {
        if (j + 1 < nslab) issue(j + 1, (j + 1) & 1, false);
        const char *sb = wait(j & 1);
        {
            int en[NB];
            slab_scales(sb, en, fsc);
            if (j > 0) {
                int d[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) d[b] = ecur[b] - en[b];
                pr_shift<NB, CT>(st, d);
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) ecur[b] = en[b];
        }
#pragma unroll
        for (int S = 0; S < M; ++S) ck[((int64_t)j * M + S) * 32 + lane] = st[S];
        const PT *sv = reinterpret_cast<const PT *>(sb);
#pragma unroll
        for (int jj = 0; jj < kPS; ++jj) {
            CT f[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = (CT)sv[(b * kPS + jj) * 32 + lane] * fsc[b];
            pr_step<NB, CT>(st, wt, f);
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // stage reads before its refill
    }
    // the checkpoints (generic stores) are read back by bulk copies (async proxy)
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncwarp();
    // ---- exchange: the other direction's state entering my half, in my last slab's scale
    CT oth[M];
#pragma unroll
    for (int S = 0; S < M; ++S) oth[S] = __shfl_xor_sync(0xffffffffu, st[S], 1);
    {
        int d[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) d[b] = __shfl_xor_sync(0xffffffffu, ecur[b], 1) - ecur[b];
        pr_shift<NB, CT>(oth, d);
    }
    // ---- phase 2: other walk from position npos-1 down to 0, own states rebuilt per slab
    PT *vo = static_cast<PT *>(pp.phit) + ((int64_t)k * pp.nblk + blk) * npos * 32 + lane;
    int *eo = pp.E + pr_xrec(pp, k, blk, 0) + lane;  // phi_k's E of slab j at eo[j * l * 64]
    const int64_t xst = (int64_t)L * 64;
    int eprev = INT_MIN;
    bool bad = false;
    const int s0 = nslab & 1;  // phase 1 left its last slab in stage (nslab - 1) & 1: start on the other
    issue(nslab - 1, s0, true);
    int t = 0;
#pragma unroll 1
    for (int j = nslab - 1; j >= 0; --j, ++t) {
        if (j > 0) issue(j - 1, (t + 1 + s0) & 1, true);
        const char *sb = wait((t + s0) & 1);
        if (j < nslab - 1) {
            // entering slab j from slab j + 1: the other direction's state into this slab's scale
            int en[NB], d[NB];
            slab_scales(sb, en, fsc);
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                d[b] = ecur[b] - en[b];
                ecur[b] = en[b];
            }
            pr_shift<NB, CT>(oth, d);
        }
        const PT *sv = reinterpret_cast<const PT *>(sb);
        const MT *sm = reinterpret_cast<const MT *>(sb + ST::OFF_MU);
        const CT *sc = reinterpret_cast<const CT *>(sb + ST::OFF_CK);
        double o[kPS];  // phi_k relative to the slab scales, normalised per slab below
#pragma unroll
        for (int sub = 1; sub >= 0; --sub) {
            // rebuild own states of positions sub*kPQ .. sub*kPQ+kPQ-1 from the slab checkpoint
            CT H[kPQ][M];
#pragma unroll
            for (int S = 0; S < M; ++S) st[S] = sc[S * 32 + lane];
#pragma unroll 1
            for (int jj = 0; jj < sub * kPQ; ++jj) {  // (rolled: bounds the live registers)
                CT f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = (CT)sv[(b * kPS + jj) * 32 + lane] * fsc[b];
                pr_step<NB, CT>(st, wt, f);
            }
#pragma unroll
            for (int i = 0; i < kPQ; ++i) {
                const int jj = sub * kPQ + i;
                CT f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = (CT)sv[(b * kPS + jj) * 32 + lane] * fsc[b];
                pr_step<NB, CT>(st, wt, f);
#pragma unroll
                for (int S = 0; S < M; ++S) H[i][S] = st[S];
            }
#pragma unroll
            for (int i = kPQ - 1; i >= 0; --i) {
                const int jj = sub * kPQ + i;
                CT hd[M];
#pragma unroll
                for (int S = 0; S < M; ++S) hd[S] = S == 0 ? oth[S] : wt[pc(S)] * oth[S];
                const CT J = pr_combine<NB, CT>(H[i], hd);
                CT f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = (CT)sv[(b * kPS + jj) * 32 + lane] * fsc[b];
#pragma unroll
                for (int S = 0; S < M; ++S) oth[S] = hd[S];
                pr_place<NB, CT>(oth, f);
                const CT mu = (CT)sm[jj * 32 + lane];
                const double q = TR::div(mu, J);
                const bool nz = TR::nz(mu);  // padding: mu = 0
                bad |= nz && !finite_positive(q);
                o[jj] = nz ? q : 0.0;
            }
        }
        // slab output: mantissas normalised to max in [1, 2), exponent E_k = -sum_b G_b + emax
        int emax = INT_MIN;
#pragma unroll
        for (int jj = 0; jj < kPS; ++jj)
            if (o[jj] != 0.0) emax = max(emax, pr_ilog2(o[jj]));
        int sumE = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b) sumE += ecur[b];
        int Ek;
        if (emax != INT_MIN) {
            Ek = -sumE + emax;
            const double sc2 = pr_pow2c(-emax);
#pragma unroll
            for (int jj = 0; jj < kPS; ++jj) o[jj] *= sc2;
        } else {
            Ek = eprev != INT_MIN ? eprev : -sumE;  // zero slab: the neighbour's exponent
        }
        if (!bad && !dead) {
#pragma unroll
            for (int jj = 0; jj < kPS; ++jj) vo[(int64_t)(j * kPS + jj) * 32] = (PT)o[jj];
            eo[j * xst] = Ek;
        }
        eprev = Ek;
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // stage reads before its refill
    }
    if constexpr (ENV) pair_envelope(eo, eo + 32, nslab, c8, xst);
    // phi_k and its exponents (generic stores) are read by the next update's bulk copies (async proxy)
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncwarp();
    return bad;
}

template <int NB, typename PT, typename MT, typename CT>
__global__ void __launch_bounds__(kPWarps * 32, 1) k_pair_sinkhorn(PairPlan pp) {
    constexpr int L = NB + 1;
    extern __shared__ __align__(16) char pr_sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kPWarps + wib;
    const int64_t nw = (int64_t)gridDim.x * kPWarps;
    char *stg = pr_sm + (size_t)wib * kPStages * PStage<NB, PT, MT, CT>::BYTES;
    __shared__ uint64_t pr_bar[kPWarps][kPStages];
    uint64_t *bar = pr_bar[wib];
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kPStages; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    unsigned par = 0;
    CT *ck = reinterpret_cast<CT *>(pp.ckpt) + gw * (int64_t)pp.nslab * (1 << NB) * 32;
    for (int64_t blk = gw; blk < pp.nblk; blk += nw) {
        const int64_t inst = blk * 16 + (lane >> 1);
        const bool active = inst < pp.batch;
        CT wt[NB + 2];  // w_a = exp(-a(l-a) h / eta) in fp64, rounded to the compute type (A15)
        double c8;      // the kernel's decay over one slab, in bits (pair_envelope)
        {
            const double eta = active ? pp.eta[inst] : 1.0;
            c8 = (double)(kPS * (L - 1)) * pp.h / eta * 1.4426950408889634;
#pragma unroll
            for (int a = 0; a <= NB + 1; ++a) wt[a] = (CT)(a <= L ? exp(-(double)(a * (L - a)) * pp.h / eta) : 0.0);
        }
        bool bad = !active;
        int fail = -1, done = 0;
        for (int t = 1; t <= pp.iters; ++t) {
            if (__all_sync(0xffffffffu, bad)) break;
            bool b2 = false;
            for (int k = 0; k < L; ++k) {
                const bool r = pair_update<NB, PT, MT, CT>(pp, blk, k, wt, stg, bar, par, ck, lane, bad, c8);
                b2 |= r && !bad;
                // the pair shares one instance: both threads see the flag before the next update
                const bool pb = __shfl_xor_sync(0xffffffffu, (int)r, 1) != 0;
                if ((r || pb) && !bad) {
                    bad = true;
                    fail = t;
                }
                __syncwarp();
            }
            if (!bad) done = t;
        }
        if (active && (lane & 1) == 0) {
            const bool failed = fail >= 0;
            pp.status[inst] = failed ? 6 : 0;
            pp.fail_iter[inst] = failed ? fail : -1;
            pp.iters_done[inst] = done;
            pp.converged[inst] = 0;
            pp.resid[inst] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
}

// ---------------------------------------------------------------------------------------
// Conversions at the API boundary.  Thread per (q, blk, slab, lane).
//   op 0: u[q] (caller layout [batch][N], LOG or LINEAR) -> mantissas + slab exponents
//   op 1: mantissas + exponents -> u[q]
//   op 2: mu[q] ([batch][N], fp64) -> this layout (MT)
// Position p of half hf -> grid point (-1: padding).  The padding sits at the OPEN end of each half
// (positions 0 .. pad-1): the own walk starts there from e_{} and a zero scaling with the identity
// diag on e_{} leaves it e_{}, so no position needs a predicate in the walks.
__device__ __forceinline__ int64_t pr_point(const PairPlan &pp, int hf, int64_t p) {
    const int64_t pad = (int64_t)pp.nslab * kPS - (hf ? pp.nB : pp.nA);
    if (p < pad) return -1;
    return hf ? pp.N - 1 - (p - pad) : p - pad;
}

template <typename PT, typename MT>
__global__ void k_pair_convert(PairPlan pp, void *const *u, int op, int log_repr) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)pp.l * pp.nblk * pp.nslab * 32;
    if (tid >= nthr) return;
    const int lane = (int)(tid & 31);
    const int64_t j = (tid >> 5) % pp.nslab;
    const int64_t blk = ((tid >> 5) / pp.nslab) % pp.nblk;
    const int q = (int)((tid >> 5) / pp.nslab / pp.nblk);
    const int hf = lane & 1;
    const int64_t inst = blk * 16 + (lane >> 1);
    const int64_t npos = (int64_t)pp.nslab * kPS;
    const int64_t vbase = (((int64_t)q * pp.nblk + blk) * npos + j * kPS) * 32 + lane;
    int *E = pp.E + pr_xrec(pp, q, blk, j) + lane;
    const bool active = inst < pp.batch;
    if (op == 2) {
        const double *src = reinterpret_cast<const double *const *>(u)[q];
        MT *dst = static_cast<MT *>(pp.mu);
        for (int jj = 0; jj < kPS; ++jj) {
            const int64_t p = j * kPS + jj;
            const int64_t x = pr_point(pp, hf, p);
            dst[vbase + jj * 32] = (MT)((active && x >= 0) ? src[inst * pp.N + x] : 0.0);
        }
        return;
    }
    PT *m = static_cast<PT *>(pp.phit);
    if (op == 1) {
        if (!active) return;
        double *dst = reinterpret_cast<double *const *>(u)[q] + inst * pp.N;
        const int e = *E;
        for (int jj = 0; jj < kPS; ++jj) {
            const int64_t p = j * kPS + jj;
            const int64_t x = pr_point(pp, hf, p);
            if (x < 0) continue;
            const double v = (double)m[vbase + jj * 32];
            dst[x] = log_repr ? (v > 0.0 ? log(v) + (double)e * 0.69314718055994530942 : -INFINITY)
                                                : (v == 0.0 ? 0.0 : ldexp(v, e));
        }
        return;
    }
    // import: the exponent of the slab (INT_MIN: no nonzero value -> fixed by k_pair_fill)
    const double *src = reinterpret_cast<const double *const *>(u)[q] + (active ? inst * pp.N : 0);
    double v[kPS];
    int emax = INT_MIN;
    for (int jj = 0; jj < kPS; ++jj) {
        const int64_t p = j * kPS + jj;
        const int64_t xi = pr_point(pp, hf, p);
        double x = (active && xi >= 0) ? src[xi] : (log_repr ? -INFINITY : 0.0);
        v[jj] = x;
        if (log_repr) {
            if (x > -INFINITY) emax = max(emax, (int)floor(x * 1.4426950408889634074));
        } else if (x > 0.0) {
            int e;
            frexp(x, &e);
            emax = max(emax, e - 1);
        }
    }
    for (int jj = 0; jj < kPS; ++jj) {
        double mm = 0.0;
        if (emax != INT_MIN) {
            if (log_repr) mm = v[jj] > -INFINITY ? exp(v[jj] - (double)emax * 0.69314718055994530942) : 0.0;
            else mm = v[jj] > 0.0 ? ldexp(v[jj], -emax) : 0.0;
        }
        m[vbase + jj * 32] = (PT)mm;
    }
    *E = emax;
}

// zero slabs (exponent INT_MIN) take the nearest previous slab's exponent (the first ones: the next
// nonzero slab's; an all-zero vector: 0).  Thread per (q, blk, lane).
__global__ void k_pair_fill(PairPlan pp) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (int64_t)pp.l * pp.nblk * 32) return;  // whole warps (the count is a multiple of 32)
    const int lane = (int)(tid & 31);
    const int q = (int)((tid >> 5) / pp.nblk);
    const int64_t blk = (tid >> 5) % pp.nblk;
    const int64_t xst = (int64_t)pp.l * 64;
    int *E = pp.E + pr_xrec(pp, q, blk, 0) + lane;
    int first = INT_MIN;
    for (int j = 0; j < pp.nslab && first == INT_MIN; ++j) first = E[j * xst];
    int prev = first == INT_MIN ? 0 : first;
    for (int j = 0; j < pp.nslab; ++j) {
        const int e = E[j * xst];
        if (e == INT_MIN) E[j * xst] = prev;
        else prev = e;
    }
    if (pp.f32c) {
        // state scales of the fp32 walks (pair_envelope)
        const int64_t inst = blk * 16 + (lane >> 1);
        const double eta = inst < pp.batch ? pp.eta[inst] : 1.0;
        const double c8 = (double)(kPS * (pp.l - 1)) * pp.h / eta * 1.4426950408889634;
        pair_envelope(E, E + 32, pp.nslab, c8, xst);
    }
}

int64_t pair_slots() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int64_t)sms * 8;
}

cudaError_t launch_pair_convert(const PairPlan &pp, void *const *u_dev, int op, int log_repr, cudaStream_t s,
                                int64_t *launches) {
    const int64_t n = (int64_t)pp.l * pp.nblk * pp.nslab * 32;
    const unsigned g = (unsigned)((n + 255) / 256);
    if (pp.f32) k_pair_convert<float, float><<<g, 256, 0, s>>>(pp, u_dev, op, log_repr);
    else k_pair_convert<double, double><<<g, 256, 0, s>>>(pp, u_dev, op, log_repr);
    ++*launches;
    if (op == 0) {
        const int64_t nf = (int64_t)pp.l * pp.nblk * 32;
        k_pair_fill<<<(unsigned)((nf + 255) / 256), 256, 0, s>>>(pp);
        ++*launches;
    }
    return cudaGetLastError();
}

template <int NB, typename PT, typename MT, typename CT>
static cudaError_t pair_go(const PairPlan &pp, cudaStream_t s) {
    const size_t sm = pair_smem<NB, PT, MT, CT>();
    smem_attr((const void *)k_pair_sinkhorn<NB, PT, MT, CT>, sm);
    const int64_t warps = std::min<int64_t>(pp.nblk, pp.slots);
    const unsigned grid = (unsigned)((warps + kPWarps - 1) / kPWarps);
    k_pair_sinkhorn<NB, PT, MT, CT><<<grid, kPWarps * 32, sm, s>>>(pp);
    return cudaGetLastError();
}

cudaError_t launch_pair_sinkhorn(const PairPlan &pp, cudaStream_t s, int64_t *launches) {
    ++*launches;
    const int NB = pp.l - 1;
    if (pp.f32 && pp.f32c) {
        switch (NB) {
            case 1: return pair_go<1, float, float, float>(pp, s);
            case 2: return pair_go<2, float, float, float>(pp, s);
            case 3: return pair_go<3, float, float, float>(pp, s);
            case 4: return pair_go<4, float, float, float>(pp, s);
        }
    } else if (pp.f32) {
        switch (NB) {
            case 1: return pair_go<1, float, float, double>(pp, s);
            case 2: return pair_go<2, float, float, double>(pp, s);
            case 3: return pair_go<3, float, float, double>(pp, s);
            case 4: return pair_go<4, float, float, double>(pp, s);
        }
    } else {
        switch (NB) {
            case 1: return pair_go<1, double, double, double>(pp, s);
            case 2: return pair_go<2, double, double, double>(pp, s);
            case 3: return pair_go<3, double, double, double>(pp, s);
            case 4: return pair_go<4, double, double, double>(pp, s);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace mmot
