// lanes.cu -- the lane-state family for l = 6 (NB = 5 bound marginals, 2^5 = 32 subset states): one
// warp per chain, lane S = subset state S.  (C3: l = 6, N = 1e5.)
//
// The two-walk family keeps a chain's 32 states (and, for the chain operators, 6 x 32 operator
// entries) in one thread; at l = 6 that is register-bound and forces chains of 8 points, so the
// operator scan over 12 500 chains (compositions of 192-entry operators) dominated the update
// (DESIGN.md §5).  Here the same recurrence (dp.cuh) runs with the state vector spread over the
// lanes of a warp:
//   diag   st[S] *= w_{|S|}                               (lane-dependent constant)
//   place  for each bound b: st[S] += f_b * st[S ^ b]      (S containing b; one shuffle + FMA)
//   combine J = sum_S F[S] H[S^c]                         (one shuffle + a warp reduction)
// and the chain operators (the extended walk of dp.cuh opx_*, slices c = 0..5) are 6 registers per
// lane.  Chains of 32 points (3 125 chains at N = 1e5) and a two-level scan:
//   k_ls_ops    warp per chain: extended operator walk -> prefix / suffix operators (OpShape layout)
//   k_ls_scan1  CTA per group of 32 chains (one warp each): Kogge-Stone over the group in shared
//               memory, compositions driven by a balanced term table (648 terms over 32 lanes);
//               stores each chain's inclusive in-group operator and the group aggregate
//   k_ls_scan2  one CTA per direction: scan of the group aggregates -> the state vector entering
//               every group (an operator applied to e_empty is its slice c = 0)
//   k_ls_apply  warp per chain: carries (in-group operator applied to the group carry), suffix walk
//               with 8-point checkpoints, prefix walk with 8-point suffix rebuild, combine, epilogue.
// Suffix direction: the same scan over the reversed chain order (the chain to the right is applied
// first).  Operators compose as C_c[V] = sum_{U in V} A_c[U] B_{c+|U|}[V \ U] (A first; dp.cuh
// op_compose) and apply as y[S] = sum_{U in S} x[U] G_{|U|}[S \ U] (op_apply).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <vector>

#include "internal.h"
#include "walk.cuh"

namespace mmot {

constexpr int kLsNB = 5;
constexpr int kLsM = 1 << kLsNB;              // 32 states = 32 lanes
constexpr int kLsSZ = (kLsNB + 1) * kLsM;     // 192 operator entries
constexpr int kLsZero = kLsSZ;                // zero slot index in shared operator buffers
constexpr int kLsStride = kLsSZ + 1;
constexpr int kLsMaxTerms = 40;                // per lane (648 terms / 32 lanes ~ 20.3 after balancing)
constexpr int kLsT = 32;                       // terms per lane after balancing (the largest destination has 32)

// identity operator (G_c[V] = [V empty]): applying it returns the state unchanged
__device__ double g_ls_ident[kLsSZ];

// composition term table: [t][lane] -> a | b << 8 | dst << 16 | flush << 24
__device__ uint32_t g_ls_tbl[kLsMaxTerms * 32];
__device__ int g_ls_nterms;

static int ls_popc(int x) { int c = 0; while (x) { c += x & 1; x >>= 1; } return c; }

cudaError_t ls_init_tables() {
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (done.count(dev)) return cudaSuccess;
    struct Dst { int dst; std::vector<std::pair<int, int>> terms; };
    std::vector<Dst> dsts;
    for (int c = 0; c <= kLsNB; ++c)
        for (int V = 0; V < kLsM; ++V) {
            if (ls_popc(V) > kLsNB - c) continue;
            Dst d{c * kLsM + V, {}};
            for (int U = 0; U < kLsM; ++U)
                if ((U & V) == U) d.terms.push_back({c * kLsM + U, (c + ls_popc(U)) * kLsM + (V ^ U)});
            dsts.push_back(d);
        }
    std::sort(dsts.begin(), dsts.end(), [](const Dst &a, const Dst &b) { return a.terms.size() > b.terms.size(); });
    std::vector<std::vector<uint32_t>> lanes(32);
    std::vector<size_t> load(32, 0);
    for (const Dst &d : dsts) {
        const int ln = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        for (size_t i = 0; i < d.terms.size(); ++i) {
            const uint32_t flush = i + 1 == d.terms.size() ? 1u : 0u;
            lanes[ln].push_back((uint32_t)d.terms[i].first | ((uint32_t)d.terms[i].second << 8) |
                                ((uint32_t)d.dst << 16) | (flush << 24));
        }
        load[ln] += d.terms.size();
    }
    const int T = (int)*std::max_element(load.begin(), load.end());
    if (T > kLsT) return cudaErrorInvalidValue;
    std::vector<uint32_t> tbl((size_t)kLsMaxTerms * 32, (uint32_t)kLsZero | ((uint32_t)kLsZero << 8));
    for (int ln = 0; ln < 32; ++ln)
        for (size_t t = 0; t < lanes[ln].size(); ++t) tbl[t * 32 + ln] = lanes[ln][t];
    std::vector<double> ident(kLsSZ, 0.0);
    for (int c = 0; c <= kLsNB; ++c) ident[(size_t)c * kLsM] = 1.0;
    cudaError_t e = cudaMemcpyToSymbol(g_ls_ident, ident.data(), ident.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_ls_tbl, tbl.data(), tbl.size() * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_ls_nterms, &T, sizeof(int));
    if (e == cudaSuccess) done.insert(dev);
    return e;
}

// This lane's terms of the composition table, loaded once per kernel into registers.


// C = compose(A first, B second) in shared memory (stride kLsStride, zero slot at kLsZero); one warp.
// Fully unrolled over the lane's terms: the shared loads of all terms are independent (only the
// accumulation chains of one destination are sequential).
extern __shared__ double ls_sm[];  // the scan kernels' dynamic shared memory (indexed, so every
                                   // access compiles to LDS / STS rather than generic loads)

__shared__ uint32_t ls_tbl_sm[kLsT * 32];  // the composition term table, staged once per CTA

// Cg = compose(A first, B second); A, B are offsets (in doubles) of operators in ls_sm, Cg a
// GLOBAL scratch operator: the result stores cannot alias the shared operand loads, so the compiler
// issues all of a lane's operand loads ahead of its accumulation chains.  The caller copies Cg back
// (after __syncwarp + __threadfence_block).
__device__ __forceinline__ double ls_lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void ls_compose_g(int A, int B, double *__restrict__ Cg) {
    const int lane = threadIdx.x & 31;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(ls_sm + A);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(ls_sm + B);
    uint32_t e[kLsT];
#pragma unroll
    for (int t = 0; t < kLsT; ++t) e[t] = ls_tbl_sm[t * 32 + lane];
    double acc = 0.0;
#pragma unroll
    for (int t0 = 0; t0 < kLsT; t0 += 16) {
        // volatile shared loads keep their program order: all 32 are issued before the FMA chains
        double a[16], b[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a[k] = ls_lds(sa + 8u * (e[t0 + k] & 0xff));
            b[k] = ls_lds(sb + 8u * ((e[t0 + k] >> 8) & 0xff));
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(a[k]), "d"(b[k]));
            if (e[t0 + k] >> 24) {
                __stcg(Cg + ((e[t0 + k] >> 16) & 0xff), acc);
                acc = 0.0;
            }
        }
    }
}

// y = G(x) for a state vector held one entry per lane (x: this lane's x[S]); G in memory (global or
// shared), OpShape layout.  Lane S sums over the subsets U of S.
__device__ __forceinline__ double ls_apply(const double *G, double x, int lane) {
    double acc = 0.0;
#pragma unroll
    for (int U = 0; U < kLsM; ++U) {
        const double xu = __shfl_sync(0xffffffffu, x, U);
        const double g = G[__popc(U) * kLsM + (lane ^ U)];
        acc = fma((U & lane) == U ? xu : 0.0, g, acc);
    }
    return acc;
}

// place_x (dp_place) on the lane-distributed state: st[S] += f_b st[S ^ b] for S containing b.
// mb[b] = 1 if b is in this lane's S, else 0 (the predicate as a multiplier: no selects).
__device__ __forceinline__ double ls_place(double st, const double (&f)[kLsNB], const double (&mb)[kLsNB]) {
#pragma unroll
    for (int b = 0; b < kLsNB; ++b) {
        const double o = __shfl_xor_sync(0xffffffffu, st, 1 << b);
        st = fma(f[b] * mb[b], o, st);
    }
    return st;
}

// Chains are kLsP = 32 points; the last chain is zero-padded beyond N (phi = 0 places nothing and
// the suffix weight of an edge right of every placed index is w_0 = 1, so padding is exact for the
// suffix direction; the last chain's prefix operator / carry-out is never used).  Fixed trip counts
// keep every shuffle warp-uniform.
constexpr int kLsP = 32;

// ---------------------------------------------------------------------------------------
// Chain operators: extended walk (dp.cuh opx_step / opx_store) with lane = V.  Entries beyond the
// extended range (c + |V| > l) are unused; their diag multiplier is 0 so they stay bounded (they
// never feed a used entry: place only moves from smaller to larger sets).
__global__ void __launch_bounds__(128) k_ls_ops(Plan p, LsWork w) {
    constexpr int NB = kLsNB, L = NB + 1, M = kLsM;
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= w.C || *p.stop) return;
    const int pcS = __popc(lane);
    const int64_t x0 = c * kLsP;
    double wl[NB + 1], mb[NB];
#pragma unroll
    for (int cc = 0; cc <= NB; ++cc) {
        const int a = cc + pcS;
        wl[cc] = a > L ? 0.0 : ((a > 0 && a < L) ? p.W.w[a] : 1.0);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) mb[b] = ((lane >> b) & 1) ? 1.0 : 0.0;
    double stg[NB];
    const int64_t xi = x0 + lane;
#pragma unroll
    for (int b = 0; b < NB; ++b) stg[b] = xi < p.N ? p.bound[b][xi] : 0.0;
    double G[NB + 1];
#pragma unroll
    for (int cc = 0; cc <= NB; ++cc) G[cc] = lane == 0 ? 1.0 : 0.0;
#pragma unroll
    for (int j = 0; j < kLsP; ++j) {
        double fm[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) fm[b] = __shfl_sync(0xffffffffu, stg[b], j) * mb[b];
        if (j > 0) {
#pragma unroll
            for (int cc = 0; cc <= NB; ++cc) G[cc] *= wl[cc];
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
#pragma unroll
            for (int cc = 0; cc <= NB; ++cc) G[cc] = fma(fm[b], __shfl_xor_sync(0xffffffffu, G[cc], 1 << b), G[cc]);
        }
    }
    // prefix operator w_c Gt_c, suffix operator w_c Gt_{l-c-|V|} (Gt_l[{}] = 1)
    double *pf = w.ops_f + c * kLsSZ, *pb = w.ops_b + c * kLsSZ;
#pragma unroll
    for (int cc = 0; cc <= NB; ++cc) {
        const bool valid = cc + pcS <= NB;
        const int cp = L - cc - pcS;
        double r = 1.0;
#pragma unroll
        for (int i = 0; i <= NB; ++i)
            if (i == cp) r = G[i];
        const double wc = cc == 0 ? 1.0 : p.W.w[cc];
        pf[cc * M + lane] = valid ? wc * G[cc] : 0.0;
        pb[cc * M + lane] = valid ? wc * r : 0.0;
    }
}

// ---------------------------------------------------------------------------------------
// Scan: a multi-level work-efficient (Blelloch) block scan over the operators, 32 items per CTA
// (one warp each), per direction (blockIdx.y; direction 1 runs over the reversed chain order).
// Level L reads the items of level L (level 0: the chain operators), writes each item's exclusive
// prefix within its block (excl: the composition of the block's earlier items) and the block
// aggregates, which are the items of level L + 1; the top level has a single block.  The carries
// then flow down: carry(item) = excl(item) applied to carry(block), with carry = e_empty above the
// top (so the top level's carries are the slice 0 of its exclusive prefixes).  Compositions read
// their term table and operands from shared memory (all accesses LDS / STS).
__device__ __forceinline__ void ls_tbl_to_smem(uint32_t *st) {
    for (int i = threadIdx.x; i < kLsT * 32; i += blockDim.x) st[i] = g_ls_tbl[i];
    __syncthreads();
}
__device__ __forceinline__ void ls_set_identity(int o, int lane) {
#pragma unroll
    for (int cc = 0; cc <= kLsNB; ++cc) ls_sm[o + cc * kLsM + lane] = lane == 0 ? 1.0 : 0.0;
    if (lane == 0) ls_sm[o + kLsZero] = 0.0;
}
__device__ __forceinline__ void ls_copy_op(int o, int in, int lane) {
#pragma unroll
    for (int cc = 0; cc <= kLsNB; ++cc) ls_sm[o + cc * kLsM + lane] = ls_sm[in + cc * kLsM + lane];
    if (lane == 0) ls_sm[o + kLsZero] = 0.0;
}
__device__ __forceinline__ void ls_store_op(double *g, int o, int lane) {
#pragma unroll
    for (int cc = 0; cc <= kLsNB; ++cc)
        g[cc * kLsM + lane] = (__popc(lane) <= kLsNB - cc) ? ls_sm[o + cc * kLsM + lane] : 0.0;
}
__device__ __forceinline__ void ls_load_op(int o, const double *g, int lane) {
#pragma unroll
    for (int cc = 0; cc <= kLsNB; ++cc) ls_sm[o + cc * kLsM + lane] = g[cc * kLsM + lane];
    if (lane == 0) ls_sm[o + kLsZero] = 0.0;
}




// in: level items in scan order ([n][192]; level 0 with rev = 1 reads chain C-1-r for item r);
// excl: [n][192] exclusive in-block prefixes; agg: [n/32][192] block aggregates (null at the top).
struct LsLevel {
    const double *in[2];
    double *excl[2];
    double *agg[2];
    double *scr;  // global scratch [2][blocks][32][192] (composition results)
    int64_t n;
    int rev1;  // direction 1 reads `in` reversed (level 0: chain order)
};

__global__ void __launch_bounds__(kLsB * 32, 1) k_ls_blockscan(LsLevel L, const int *stop) {
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int dir = blockIdx.y;
    const int64_t item = (int64_t)blockIdx.x * kLsB + wi;
    if (*stop) return;
    ls_tbl_to_smem(ls_tbl_sm);
    const int me = wi * kLsStride;
    double *cg = L.scr + (((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kLsB + wi) * kLsSZ;
    if (item < L.n) {
        const int64_t src = (dir == 1 && L.rev1) ? L.n - 1 - item : item;
        ls_load_op(me, L.in[dir] + src * kLsSZ, lane);
    } else {
        ls_set_identity(me, lane);
    }
    __syncthreads();
    // up-sweep: buf[w] <- compose(buf[w - d], buf[w]) for w = 2d-1, 4d-1, ...
    for (int d = 1; d < kLsB; d <<= 1) {
        if (((wi + 1) & (2 * d - 1)) == 0) {
            ls_compose_g(me - d * kLsStride, me, cg);
            __syncwarp();
            __threadfence_block();
            ls_load_op(me, cg, lane);
        }
        __syncthreads();
    }
    if (wi == kLsB - 1) {
        if (L.agg[dir]) ls_store_op(L.agg[dir] + (int64_t)blockIdx.x * kLsSZ, me, lane);
        __syncwarp();
        ls_set_identity(me, lane);
    }
    __syncthreads();
    // down-sweep: (left, right) <- (right, compose(right, left)) -- the parent's prefix first
    for (int d = kLsB / 2; d >= 1; d >>= 1) {
        if (((wi + 1) & (2 * d - 1)) == 0) {
            const int left = me - d * kLsStride;
            ls_compose_g(me, left, cg);
            __syncwarp();
            __threadfence_block();
            ls_copy_op(left, me, lane);
            __syncwarp();
            ls_load_op(me, cg, lane);
        }
        __syncthreads();
    }
    if (item < L.n) ls_store_op(L.excl[dir] + item * kLsSZ, me, lane);
}

// carry[item] = excl[item](carry_parent[item / 32]) (e_empty above the top level), per direction.
__global__ void __launch_bounds__(128) k_ls_down(const double *excl0, const double *excl1, const double *par0,
                                                 const double *par1, double *car0, double *car1, int64_t n,
                                                 const int *stop) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= 2 * n || *stop) return;
    const int dir = gw >= n;
    const int64_t item = dir ? gw - n : gw;
    const double *ex = (dir ? excl1 : excl0) + item * kLsSZ;
    const double *par = dir ? par1 : par0;
    const double x = par ? par[(item / kLsB) * kLsM + lane] : (lane == 0 ? 1.0 : 0.0);
    (dir ? car1 : car0)[item * kLsM + lane] = ls_apply(ex, x, lane);
}

// ---------------------------------------------------------------------------------------
// Apply: warp per chain.  MODE_UPD: phi_k <- mu_k / J_k; MODE_MARG: out = phi_k J_k; MODE_RES:
// partial[c] = sum |phi_k J_k - mu_k|.  Points beyond N (the last chain's padding) hold phi = 0.
template <int MODE>
__global__ void __launch_bounds__(128) k_ls_apply(Plan p, LsWork w) {
    constexpr int NB = kLsNB, M = kLsM;
    constexpr int Q = 8;              // checkpoint block
    constexpr int NQ = kLsP / Q;
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= w.C || *p.stop) return;
    const int pcS = __popc(lane);
    const int64_t x0 = c * kLsP;
    const double wl = lane == 0 ? 1.0 : p.W.w[pcS];  // diag weight of state S (w_0 = 1)
    double mb[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) mb[b] = ((lane >> b) & 1) ? 1.0 : 0.0;
    // carries: prefix state entering the chain, suffix state after its last point
    // carries (level 0 of the scan, in scan order: direction 1 is reversed)
    double F = w.lv_car[0][0][c * M + lane], B = w.lv_car[0][1][(w.C - 1 - c) * M + lane];
    // the chain's bound values in registers (lane j: point x0 + j), padded with zeros beyond N
    double stg[NB];
    const int64_t xi = x0 + lane;
    const bool in = xi < p.N;
#pragma unroll
    for (int b = 0; b < NB; ++b) stg[b] = in ? p.bound[b][xi] : 0.0;
    const double vmu = (MODE == MODE_UPD || MODE == MODE_RES) && in ? p.muk[xi] : 0.0;
    const double vph = (MODE == MODE_MARG || MODE == MODE_RES) && in ? p.phik[xi] : 0.0;
    // walk 1 (right to left): checkpoints ck[q] = B at x0 + Q (q+1)
    double ck[NQ];
#pragma unroll
    for (int q = NQ - 1; q >= 0; --q) {   // (ck needs compile-time indices: unrolled, 3 x 8 points)
        ck[q] = B;
        if (q > 0) {
#pragma unroll
            for (int m = Q - 1; m >= 0; --m) {
                double f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = __shfl_sync(0xffffffffu, stg[b], q * Q + m);
                B *= wl;                   // edge (m, m+1)
                B = ls_place(B, f, mb);
            }
        }
    }
    // walk 2 (left to right): rebuild the Q suffix states of each block, prefix step, combine
    double tj = 0.0;  // J of this lane's point (lane j <-> x0 + j), selected without branches
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) {
        double H[Q];
        double st = q == 0 ? ck[0] : q == 1 ? ck[1] : q == 2 ? ck[2] : ck[3];
#pragma unroll
        for (int i = Q - 1; i >= 0; --i) {
            st *= wl;                      // H_m = D B_{m+1}
            H[i] = st;
            if (i > 0) {
                double f[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) f[b] = __shfl_sync(0xffffffffu, stg[b], q * Q + i);
                st = ls_place(st, f, mb);
            }
        }
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int m = q * Q + i;
            double f[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = __shfl_sync(0xffffffffu, stg[b], m);
            F *= wl;
            F = ls_place(F, f, mb);
            double t = F * __shfl_xor_sync(0xffffffffu, H[i], M - 1);  // F[S] H[S^c]
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
            tj = lane == m ? t : tj;
        }
    }
    bool bad = false;
    double acc = 0.0, o_mine = 0.0;
    if (MODE == MODE_UPD) {
        const double qv = div_nr1(vmu, tj);
        const bool nz = nonzero(vmu);
        bad = nz && !finite_positive(qv);
        o_mine = nz ? qv : 0.0;
    } else if (MODE == MODE_MARG) {
        bad = vph > 0.0 && !finite_positive(tj);
        o_mine = vph * tj;
    } else {
        bad = vph > 0.0 && !finite_positive(tj);
        acc = in ? fabs(vph * tj - vmu) : 0.0;
    }
    if (MODE == MODE_UPD || MODE == MODE_MARG) {
        if (in) p.outk[xi] = o_mine;
    } else {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
        if (lane == 0) p.partial[c] = acc;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) {
        if (atomicCAS(p.status, 0, 6) == 0) *p.fail_iter = p.sweep ? *p.sweep + 1 : p.iter;
        *(volatile int *)p.stop = 1;
    }
}

cudaError_t launch_ls_product(const Plan &p, const LsWork &w, int mode, cudaStream_t s, int64_t *launches) {
    cudaError_t e = ls_init_tables();
    if (e != cudaSuccess) return e;
    const unsigned wb = (unsigned)((w.C + 3) / 4);
    k_ls_ops<<<wb, 128, 0, s>>>(p, w);
    int nl = 0;
    const size_t smb = kLsB * (size_t)kLsStride * sizeof(double);
    smem_attr((const void *)k_ls_blockscan, smb);
    // up: level 0 = chains (direction 1 reversed), then block aggregates until one block remains
    for (int lv = 0; lv < w.nlev; ++lv) {
        LsLevel L{};
        L.n = w.lv_n[lv];
        L.rev1 = lv == 0;
        L.in[0] = lv == 0 ? w.ops_f : w.lv_agg[lv - 1][0];
        L.in[1] = lv == 0 ? w.ops_b : w.lv_agg[lv - 1][1];
        L.excl[0] = w.lv_excl[lv][0];
        L.excl[1] = w.lv_excl[lv][1];
        L.agg[0] = lv + 1 < w.nlev ? w.lv_agg[lv][0] : nullptr;
        L.agg[1] = lv + 1 < w.nlev ? w.lv_agg[lv][1] : nullptr;
        L.scr = w.scr;
        k_ls_blockscan<<<dim3((unsigned)((L.n + kLsB - 1) / kLsB), 2), kLsB * 32, smb, s>>>(L, p.stop);
        ++nl;
    }
    // down: carries of every level from the top; level 0's are the chain carries (scan order)
    for (int lv = w.nlev - 1; lv >= 0; --lv) {
        const int64_t n = w.lv_n[lv];
        const double *par0 = lv + 1 < w.nlev ? w.lv_car[lv + 1][0] : nullptr;
        const double *par1 = lv + 1 < w.nlev ? w.lv_car[lv + 1][1] : nullptr;
        k_ls_down<<<(unsigned)((2 * n + 3) / 4), 128, 0, s>>>(w.lv_excl[lv][0], w.lv_excl[lv][1], par0, par1,
                                                             w.lv_car[lv][0], w.lv_car[lv][1], n, p.stop);
        ++nl;
    }
    switch (mode) {
        case MODE_UPD: k_ls_apply<MODE_UPD><<<wb, 128, 0, s>>>(p, w); break;
        case MODE_MARG: k_ls_apply<MODE_MARG><<<wb, 128, 0, s>>>(p, w); break;
        default: k_ls_apply<MODE_RES><<<wb, 128, 0, s>>>(p, w); break;
    }
    *launches += 2 + nl;
    return cudaGetLastError();
}

}  // namespace mmot
