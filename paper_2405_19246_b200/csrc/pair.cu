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
// floor(log2 x) of a positive normal double; INT_MIN for 0 / denormals
__device__ __forceinline__ int pr_ilog2(double x) {
    const int e = (int)((__double_as_longlong(x) >> 52) & 0x7ff);
    return e == 0 ? INT_MIN : e - 1023;
}

// st[S] *= 2^{sum_{b in S} d[b]}.  Neighbouring slabs' exponents differ by a few bits, so the
// usual path forms 2^{d_b} once and the 2^NB subset factors by products (exact: every partial sum
// stays inside the normal range); larger jumps take two clamped factors per state (exact for
// |n| <= 2044).
template <int NB>
__device__ __forceinline__ void pr_shift(double (&st)[1 << NB], const int (&d)[NB]) {
    constexpr int M = 1 << NB;
    bool small = true;
#pragma unroll
    for (int b = 0; b < NB; ++b) small &= d[b] >= -255 && d[b] <= 255;
    if (small) {
        double fb[NB], fac[M];
#pragma unroll
        for (int b = 0; b < NB; ++b) fb[b] = __longlong_as_double((long long)(d[b] + 1023) << 52);
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
        st[S] = (st[S] * pr_pow2c(h1)) * pr_pow2c(n - h1);
    }
}

// Shared-memory stage of one slab: bound mantissas [NB][kPS][32] (PT), mu [kPS][32] (MT),
// checkpoint [M][32] (double) -- each tile one contiguous range of global memory.
template <int NB, typename PT, typename MT>
struct PStage {
    static constexpr int M = 1 << NB;
    static constexpr int TILE_P = kPS * 32 * (int)sizeof(PT);  // one vector's slab: contiguous in global
    static constexpr int TILE_M = kPS * 32 * (int)sizeof(MT);
    static constexpr int TILE_C = M * 32 * 8;                   // the slab's checkpoint
    static constexpr int OFF_MU = NB * TILE_P;
    static constexpr int OFF_CK = OFF_MU + TILE_M;
    static constexpr int BYTES = OFF_CK + TILE_C;
};

template <int NB, typename PT, typename MT>
size_t pair_smem() {
    return (size_t)kPWarps * kPStages * PStage<NB, PT, MT>::BYTES;
}

// One Gauss-Seidel update phi_k <- mu_k / J_k of the warp's 16 instances.
template <int NB, typename PT, typename MT>
__device__ __forceinline__ bool pair_update(const PairPlan &pp, int64_t blk, int k, const double (&wt)[NB + 2],
                                            char *stg, uint64_t *bar, unsigned &par, double *ck, int lane, bool dead) {
    using ST = PStage<NB, PT, MT>;
    constexpr int L = NB + 1, M = 1 << NB;
    const int nslab = pp.nslab;
    const int64_t npos = (int64_t)nslab * kPS;
    const PT *phit = static_cast<const PT *>(pp.phit);
    const PT *vb[NB];
    const int *eb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int q = (k + 1 + b) % L;
        vb[b] = phit + ((int64_t)q * pp.nblk + blk) * npos * 32 + lane;
        eb[b] = pp.E + ((int64_t)q * pp.nblk + blk) * nslab * 32 + lane;
    }
    // one slab into stage `slot`: bulk copies issued by lane 0, completion on the slot's mbarrier
    // (the tiles are contiguous in global memory: [position][lane] and [state][lane])
    const PT *vbase[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) vbase[b] = vb[b] - lane;
    auto issue = [&](int j, int slot, bool p2) {
        if (lane == 0) {
            char *sb = stg + slot * ST::BYTES;
            mbar_arrive_expect_tx(&bar[slot], (uint32_t)(NB * ST::TILE_P + (p2 ? ST::TILE_M + ST::TILE_C : 0)));
#pragma unroll
            for (int b = 0; b < NB; ++b)
                bulk_g2s(sb + b * ST::TILE_P, vbase[b] + (int64_t)j * kPS * 32, ST::TILE_P, &bar[slot]);
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
    // ---- phase 1: own walk over positions 0 .. npos-1, checkpoint before every slab
    double st[M];
    vec_unit<NB, double>(st);
    int ecur[NB], enx[NB];  // exponents of the current slab / of the next one (loaded a slab ahead)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        ecur[b] = eb[b][0];
        enx[b] = nslab > 1 ? eb[b][32] : ecur[b];
    }
    issue(0, 0, false);
#pragma unroll 1
    for (int j = 0; j < nslab; ++j) {
        if (j > 0) {
            int d[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                d[b] = ecur[b] - enx[b];
                ecur[b] = enx[b];
                if (j + 1 < nslab) enx[b] = eb[b][(j + 1) * 32];
            }
            pr_shift<NB>(st, d);
        }
        if (j + 1 < nslab) issue(j + 1, (j + 1) & 1, false);
#pragma unroll
        for (int S = 0; S < M; ++S) ck[((int64_t)j * M + S) * 32 + lane] = st[S];
        const PT *sv = reinterpret_cast<const PT *>(wait(j & 1));
#pragma unroll
        for (int jj = 0; jj < kPS; ++jj) {
            double f[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = (double)sv[(b * kPS + jj) * 32 + lane];
            dp_diag<NB, double, true>(st, wt);
            dp_place<NB, double>(st, f);
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // stage reads before its refill
    }
    // the checkpoints (generic stores) are read back by bulk copies (async proxy)
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncwarp();
    // ---- exchange: the other direction's state entering my half, in my last slab's scale
    double oth[M];
#pragma unroll
    for (int S = 0; S < M; ++S) oth[S] = __shfl_xor_sync(0xffffffffu, st[S], 1);
    {
        int d[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) d[b] = __shfl_xor_sync(0xffffffffu, ecur[b], 1) - ecur[b];
        pr_shift<NB>(oth, d);
    }
    // ---- phase 2: other walk from position npos-1 down to 0, own states rebuilt per slab
    PT *vo = static_cast<PT *>(pp.phit) + ((int64_t)k * pp.nblk + blk) * npos * 32 + lane;
    int *eo = pp.E + ((int64_t)k * pp.nblk + blk) * nslab * 32 + lane;
    int eprev = INT_MIN;
    bool bad = false;
    const int s0 = nslab & 1;  // phase 1 left its last slab in stage (nslab - 1) & 1: start on the other
    issue(nslab - 1, s0, true);
    int t = 0;
#pragma unroll 1
    for (int j = nslab - 1; j >= 0; --j, ++t) {
        if (j > 0) {
            issue(j - 1, (t + 1 + s0) & 1, true);
#pragma unroll
            for (int b = 0; b < NB; ++b) enx[b] = eb[b][(j - 1) * 32];
        }
        const char *sb = wait((t + s0) & 1);
        const PT *sv = reinterpret_cast<const PT *>(sb);
        const MT *sm = reinterpret_cast<const MT *>(sb + ST::OFF_MU);
        const double *sc = reinterpret_cast<const double *>(sb + ST::OFF_CK);
        double o[kPS];
#pragma unroll
        for (int sub = 1; sub >= 0; --sub) {
            // rebuild own states of positions sub*kPQ .. sub*kPQ+kPQ-1 from the slab checkpoint
            double H[kPQ][M];
#pragma unroll
            for (int S = 0; S < M; ++S) st[S] = sc[S * 32 + lane];
#pragma unroll 1
            for (int jj = 0; jj < sub * kPQ; ++jj) {  // (rolled: bounds the live registers)
                double f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = (double)sv[(b * kPS + jj) * 32 + lane];
                dp_diag<NB, double, true>(st, wt);
                dp_place<NB, double>(st, f);
            }
#pragma unroll
            for (int i = 0; i < kPQ; ++i) {
                const int jj = sub * kPQ + i;
                double f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = (double)sv[(b * kPS + jj) * 32 + lane];
                dp_diag<NB, double, true>(st, wt);
                dp_place<NB, double>(st, f);
#pragma unroll
                for (int S = 0; S < M; ++S) H[i][S] = st[S];
            }
#pragma unroll
            for (int i = kPQ - 1; i >= 0; --i) {
                const int jj = sub * kPQ + i;
                double hd[M];
#pragma unroll
                for (int S = 0; S < M; ++S) hd[S] = S == 0 ? oth[S] : wt[pc(S)] * oth[S];
                const double J = combine<NB, double>(H[i], hd);
                double f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = (double)sv[(b * kPS + jj) * 32 + lane];
#pragma unroll
                for (int S = 0; S < M; ++S) oth[S] = hd[S];
                dp_place<NB, double>(oth, f);
                const double mu = (double)sm[jj * 32 + lane];
                const double q = div_nr1(mu, J);
                const bool nz = nonzero(mu);  // padding: mu = 0
                bad |= nz && !finite_positive(q);
                o[jj] = nz ? q : 0.0;
            }
        }
        // slab output: mantissas normalised to max in [1, 2), exponent E_k = -sum_b E_b + emax
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
            eo[j * 32] = Ek;
        }
        eprev = Ek;
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // stage reads before its refill
        if (j > 0) {
            int d[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                d[b] = ecur[b] - enx[b];
                ecur[b] = enx[b];
            }
            pr_shift<NB>(oth, d);
        }
    }
    // phi_k (generic stores) is read by the next update's bulk copies (async proxy)
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncwarp();
    return bad;
}

template <int NB, typename PT, typename MT>
__global__ void __launch_bounds__(kPWarps * 32, 1) k_pair_sinkhorn(PairPlan pp) {
    constexpr int L = NB + 1;
    extern __shared__ __align__(16) char pr_sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kPWarps + wib;
    const int64_t nw = (int64_t)gridDim.x * kPWarps;
    char *stg = pr_sm + (size_t)wib * kPStages * PStage<NB, PT, MT>::BYTES;
    __shared__ uint64_t pr_bar[kPWarps][kPStages];
    uint64_t *bar = pr_bar[wib];
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < kPStages; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    unsigned par = 0;
    double *ck = pp.ckpt + gw * (int64_t)pp.nslab * (1 << NB) * 32;
    for (int64_t blk = gw; blk < pp.nblk; blk += nw) {
        const int64_t inst = blk * 16 + (lane >> 1);
        const bool active = inst < pp.batch;
        double wt[NB + 2];
        {
            const double eta = active ? pp.eta[inst] : 1.0;
#pragma unroll
            for (int a = 0; a <= NB + 1; ++a) wt[a] = a <= L ? exp(-(double)(a * (L - a)) * pp.h / eta) : 0.0;
        }
        bool bad = !active;
        int fail = -1, done = 0;
        for (int t = 1; t <= pp.iters; ++t) {
            if (__all_sync(0xffffffffu, bad)) break;
            bool b2 = false;
            for (int k = 0; k < L; ++k) {
                const bool r = pair_update<NB, PT, MT>(pp, blk, k, wt, stg, bar, par, ck, lane, bad);
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
    int *E = pp.E + (((int64_t)q * pp.nblk + blk) * pp.nslab + j) * 32 + lane;
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
    if (tid >= (int64_t)pp.l * pp.nblk * 32) return;
    const int lane = (int)(tid & 31);
    int *E = pp.E + (tid >> 5) * pp.nslab * 32 + lane;
    int first = INT_MIN;
    for (int j = 0; j < pp.nslab && first == INT_MIN; ++j) first = E[j * 32];
    int prev = first == INT_MIN ? 0 : first;
    for (int j = 0; j < pp.nslab; ++j) {
        const int e = E[j * 32];
        if (e == INT_MIN) E[j * 32] = prev;
        else prev = e;
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

template <int NB, typename PT, typename MT>
static cudaError_t pair_go(const PairPlan &pp, cudaStream_t s) {
    const size_t sm = pair_smem<NB, PT, MT>();
    smem_attr((const void *)k_pair_sinkhorn<NB, PT, MT>, sm);
    const int64_t warps = std::min<int64_t>(pp.nblk, pp.slots);
    const unsigned grid = (unsigned)((warps + kPWarps - 1) / kPWarps);
    k_pair_sinkhorn<NB, PT, MT><<<grid, kPWarps * 32, sm, s>>>(pp);
    return cudaGetLastError();
}

cudaError_t launch_pair_sinkhorn(const PairPlan &pp, cudaStream_t s, int64_t *launches) {
    ++*launches;
    const int NB = pp.l - 1;
    if (pp.f32) {
        switch (NB) {
            case 1: return pair_go<1, float, float>(pp, s);
            case 2: return pair_go<2, float, float>(pp, s);
            case 3: return pair_go<3, float, float>(pp, s);
            case 4: return pair_go<4, float, float>(pp, s);
        }
    } else {
        switch (NB) {
            case 1: return pair_go<1, double, double>(pp, s);
            case 2: return pair_go<2, double, double>(pp, s);
            case 3: return pair_go<3, double, double>(pp, s);
            case 4: return pair_go<4, double, double>(pp, s);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace mmot
