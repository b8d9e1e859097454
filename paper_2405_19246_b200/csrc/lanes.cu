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
// lane.  Chains of 32 points (3 125 chains at N = 1e5) and a multi-level scan:
//   k_ls_ops    warp per chain: extended operator walk -> prefix / suffix operators (OpShape layout)
//   k_ls_blockscan  per level, CTA per block of 16 items (one warp each): Kogge-Stone over the block
//               in shared memory (two buffers), compositions driven by a balanced term table (648
//               terms over 32 lanes); stores each item's exclusive in-block prefix and the block
//               aggregate (the items of the next level)
//   k_ls_down   per level, top first: carry(item) = excl(item) applied to carry(block) (an operator
//               applied to e_empty is its slice c = 0)
//   k_ls_apply  warp per chain: carries (in-group operator applied to the group carry), suffix walk
//               with 8-point checkpoints, prefix walk with 8-point suffix rebuild, combine, epilogue.
// Suffix direction: the same scan over the reversed chain order (the chain to the right is applied
// first).  Operators compose as C_c[V] = sum_{U in V} A_c[U] B_{c+|U|}[V \ U] (A first; dp.cuh
// op_compose) and apply as y[S] = sum_{U in S} x[U] G_{|U|}[S \ U] (op_apply).
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

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
constexpr int kLsSplit = kLsSZ + 1;            // scratch slot: second half of the split destination
constexpr int kLsStride = kLsSZ + 2;
constexpr int kLsMaxTerms = 40;                // per lane (648 terms / 32 lanes ~ 20.3 after balancing)
constexpr int kLsT = 24;                       // term slots per lane after balancing (multiple of 8)
constexpr int kLsBig = kLsNB;                  // C_0[all bounds] (32 terms) is split into two 16-term halves

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
            if (c == 0 && V == kLsM - 1) {
                // the only 32-term destination: two halves, the second summed into the scratch slot
                // and added by ls_fix_split after the composition (keeps every lane at <= kLsT terms)
                Dst h{kLsSplit, std::vector<std::pair<int, int>>(d.terms.begin() + 16, d.terms.end())};
                d.terms.resize(16);
                dsts.push_back(h);
            }
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


extern __shared__ double ls_sm[];  // the scan kernels' dynamic shared memory (indexed, so every
                                   // access compiles to LDS / STS rather than generic loads)

__shared__ uint32_t ls_tbl_sm[kLsT * 32];  // the composition term table, staged once per CTA

__device__ __forceinline__ double ls_lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
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
    __shared__ double fsm[4][NB][kLsP];  // the chain's bound values (broadcast loads)
    double (*fw)[kLsP] = fsm[(threadIdx.x >> 5) & 3];
    const int64_t xi = x0 + lane;
#pragma unroll
    for (int b = 0; b < NB; ++b) fw[b][lane] = xi < p.N ? p.bound[b][xi] : 0.0;
    __syncwarp();
    double G[NB + 1];
#pragma unroll
    for (int cc = 0; cc <= NB; ++cc) G[cc] = lane == 0 ? 1.0 : 0.0;
#pragma unroll
    for (int j = 0; j < kLsP; ++j) {
        double fm[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) fm[b] = fw[b][j] * mb[b];
        if (j > 0) {
#pragma unroll
            for (int cc = 0; cc <= NB; ++cc) G[cc] *= wl[cc];
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
#pragma unroll
            for (int cc = 0; cc < NB; ++cc) G[cc] = fma(fm[b], __shfl_xor_sync(0xffffffffu, G[cc], 1 << b), G[cc]);
        }
        // slice NB: entries in range are V = {} and V = {b} (c + |V| <= l), and place never changes
        // G[{}], so G_NB[{b}] += f_b G_NB[{}] (the other lanes are out of range: diag 0 each step)
        {
            const double g0 = __shfl_sync(0xffffffffu, G[NB], 0);
            double fs = 0.0;
#pragma unroll
            for (int b = 0; b < NB; ++b) fs += fm[b];
            G[NB] = fma(fs, g0, G[NB]);
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
// Scan: a multi-level block scan over the operators, kLsB = 16 items per CTA
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
    int64_t n;
    int rev1;  // direction 1 reads `in` reversed (level 0: chain order)
    double *car[2];  // top level only (k_ls_prefix_red): carries = excl applied to e_empty; else null
};

// Kogge-Stone over the kLsB items of a block (log2 kLsB = 4 dependent compositions instead of the
// 2 log2 kLsB of a work-efficient tree), ping-ponging between two shared buffers: step d writes
// buf[s^1][w] = compose(buf[s][w - d], buf[s][w]) (w >= d) or copies buf[s][w], so every
// composition reads one buffer and stores into the other (no global round trip, no aliasing).
__device__ __forceinline__ void ls_sts(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v));
}
// C = compose(A first, B second), A, B, C offsets (doubles) in ls_sm; C must not overlap A or B.
__device__ __forceinline__ void ls_compose_s(int A, int B, int C) {
    constexpr int TB = 8;  // terms per batch (kLsT % TB == 0): table entries, then all operand loads, then the FMAs
    const int lane = threadIdx.x & 31;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(ls_sm + A);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(ls_sm + B);
    const uint32_t sc = (uint32_t)__cvta_generic_to_shared(ls_sm + C);
    double acc = 0.0;
#pragma unroll
    for (int t0 = 0; t0 < kLsT; t0 += TB) {
        uint32_t e[TB];
        double a[TB], b[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) e[k] = ls_tbl_sm[(t0 + k) * 32 + lane];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
            a[k] = ls_lds(sa + 8u * (e[k] & 0xff));
            b[k] = ls_lds(sb + 8u * ((e[k] >> 8) & 0xff));
        }
#pragma unroll
        for (int k = 0; k < TB; ++k) {
            asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(a[k]), "d"(b[k]));
            if (e[k] >> 24) {
                ls_sts(sc + 8u * ((e[k] >> 16) & 0xff), acc);
                acc = 0.0;
            }
        }
    }
    __syncwarp();
    if (lane == 0) ls_sts(sc + 8u * (kLsM - 1), ls_lds(sc + 8u * (kLsM - 1)) + ls_lds(sc + 8u * kLsSplit));
}

// TREE = false: Kogge-Stone (depth log2 kLsB, 49 compositions per block; the upper levels, where a
// few CTAs run alone and latency decides); TREE = true: work-efficient up / down sweep (depth
// 2 log2 kLsB, 30 compositions; level 0, where hundreds of CTAs share the SMs' shared-memory
// bandwidth), its results staged in the second buffer and copied back by the composing warp.
template <bool TREE>
__global__ void __launch_bounds__(kLsB * 32, 2) k_ls_blockscan(LsLevel L, const int *stop) {
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int dir = blockIdx.y;
    const int64_t item = (int64_t)blockIdx.x * kLsB + wi;
    if (*stop) return;
    ls_tbl_to_smem(ls_tbl_sm);
    const int buf = kLsB * kLsStride;  // offset of the second buffer
    const int me = wi * kLsStride;
    const double *in = dir ? L.in[1] : L.in[0];
    if (item < L.n) {
        const int64_t src = (dir == 1 && L.rev1) ? L.n - 1 - item : item;
        ls_load_op(me, in + src * kLsSZ, lane);
    } else {
        ls_set_identity(me, lane);
    }
    if (lane == 0) ls_sm[buf + me + kLsZero] = 0.0;
    __syncthreads();
    double *ex = dir ? L.excl[1] : L.excl[0];
    double *ag = dir ? L.agg[1] : L.agg[0];
    if (TREE) {
        // up-sweep: buf[w] <- compose(buf[w - d], buf[w]) for w = 2d-1, 4d-1, ...
#pragma unroll
        for (int d = 1; d < kLsB; d <<= 1) {
            if (((wi + 1) & (2 * d - 1)) == 0) {
                ls_compose_s(me - d * kLsStride, me, buf + me);
                __syncwarp();
                ls_copy_op(me, buf + me, lane);
            }
            __syncthreads();
        }
        if (wi == kLsB - 1) {
            if (ag) ls_store_op(ag + (int64_t)blockIdx.x * kLsSZ, me, lane);
            __syncwarp();
            ls_set_identity(me, lane);
        }
        __syncthreads();
        // down-sweep: (left, right) <- (right, compose(right, left)) -- the parent's prefix first
#pragma unroll
        for (int d = kLsB / 2; d >= 1; d >>= 1) {
            if (((wi + 1) & (2 * d - 1)) == 0) {
                const int left = me - d * kLsStride;
                ls_compose_s(me, left, buf + me);
                __syncwarp();
                ls_copy_op(left, me, lane);
                ls_copy_op(me, buf + me, lane);
            }
            __syncthreads();
        }
        if (item < L.n) ls_store_op(ex + item * kLsSZ, me, lane);
        return;
    }
    int cur = 0;
#pragma unroll
    for (int d = 1; d < kLsB; d <<= 1) {
        const int src = cur, dst = cur ^ buf;
        if (wi >= d) ls_compose_s(src + me - d * kLsStride, src + me, dst + me);
        else ls_copy_op(dst + me, src + me, lane);
        cur = dst;
        __syncthreads();
    }
    // cur holds the inclusive in-block prefixes; exclusive = the previous item's inclusive
    if (item < L.n) {
        if (wi == 0) {
#pragma unroll
            for (int cc = 0; cc <= kLsNB; ++cc) ex[item * kLsSZ + cc * kLsM + lane] = lane == 0 ? 1.0 : 0.0;
        } else {
            ls_store_op(ex + item * kLsSZ, cur + me - kLsStride, lane);
        }
    }
    if (wi == kLsB - 1 && ag) ls_store_op(ag + (int64_t)blockIdx.x * kLsSZ, cur + me, lane);
}

// Upper levels (a few hundred items at most): one CTA per OUTPUT instead of per block.  CTA j < n
// reduces the items of j's block before j (its exclusive in-block prefix), CTA n + b the whole block
// b (the aggregate, when the level has a parent); each by a pairwise tree of depth <= log2 kLsB in
// its own shared memory.  About 2.5x the compositions of a block scan, but spread over the GPU's
// SMs instead of 16 warps on one SM, so the level costs one tree depth of latency.
__global__ void __launch_bounds__(kLsB * 32, 2) k_ls_prefix_red(LsLevel L, const int *stop) {
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int dir = blockIdx.y;
    const int64_t j = blockIdx.x;
    if (*stop) return;
    int64_t first, cnt;
    if (j < L.n) {
        first = (j / kLsB) * kLsB;
        cnt = j - first;
    } else {
        first = (j - L.n) * kLsB;
        cnt = L.n - first < kLsB ? L.n - first : kLsB;
    }
    ls_tbl_to_smem(ls_tbl_sm);
    const int buf = kLsB * kLsStride;
    const int me = wi * kLsStride;
    const double *in = dir ? L.in[1] : L.in[0];
    if (wi < cnt) {
        const int64_t it = first + wi;
        const int64_t src = (dir == 1 && L.rev1) ? L.n - 1 - it : it;
        ls_load_op(me, in + src * kLsSZ, lane);
    } else if (wi == 0) {
        ls_set_identity(me, lane);
    }
    if (lane == 0) ls_sm[buf + me + kLsZero] = 0.0;
    __syncthreads();
#pragma unroll
    for (int d = 1; d < kLsB; d <<= 1) {
        if ((wi & (2 * d - 1)) == 0 && wi + d < cnt) {
            ls_compose_s(me, me + d * kLsStride, buf + me);
            __syncwarp();
            ls_copy_op(me, buf + me, lane);
        }
        __syncthreads();
    }
    if (wi == 0) {
        if (j < L.n) ls_store_op((dir ? L.excl[1] : L.excl[0]) + j * kLsSZ, 0, lane);
        else ls_store_op((dir ? L.agg[1] : L.agg[0]) + (j - L.n) * kLsSZ, 0, lane);
        // top level: the state entering item j is its exclusive prefix applied to e_empty, i.e. the
        // operator's slice c = 0 (the top level's k_ls_down, fused)
        if (j < L.n && L.car[0]) (dir ? L.car[1] : L.car[0])[j * kLsM + lane] = ls_sm[lane];
    }
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
__global__ void __launch_bounds__(128) k_ls_apply(Plan p, LsWork w, int fuse1) {
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
    // (level 0 of the down pass, fused here: the chain's exclusive in-block prefix applied to the
    // state entering its block; e_empty when the scan has a single level)
    const int64_t rb = w.C - 1 - c;
    double pf0, pb0;
    if (fuse1) {
        // level 1 of the down pass fused here too (scans of >= 3 levels): the block's exclusive
        // prefix at level 1 applied to the state entering its level-2 parent
        const int64_t i1f = c / kLsB, i1b = rb / kLsB;
        pf0 = ls_apply(w.lv_excl[1][0] + i1f * kLsSZ, w.lv_car[2][0][(i1f / kLsB) * M + lane], lane);
        pb0 = ls_apply(w.lv_excl[1][1] + i1b * kLsSZ, w.lv_car[2][1][(i1b / kLsB) * M + lane], lane);
    } else {
        pf0 = w.nlev > 1 ? w.lv_car[1][0][(c / kLsB) * M + lane] : (lane == 0 ? 1.0 : 0.0);
        pb0 = w.nlev > 1 ? w.lv_car[1][1][(rb / kLsB) * M + lane] : (lane == 0 ? 1.0 : 0.0);
    }
    double F = ls_apply(w.lv_excl[0][0] + c * kLsSZ, pf0, lane);
    double B = ls_apply(w.lv_excl[0][1] + rb * kLsSZ, pb0, lane);
    // the chain's bound values (lane j: point x0 + j), padded with zeros beyond N, staged in shared
    // memory: f_b at a point is then one broadcast load instead of two shuffles
    __shared__ double fsm[4][NB][kLsP];
    double (*fw)[kLsP] = fsm[(threadIdx.x >> 5) & 3];
    const int64_t xi = x0 + lane;
    const bool in = xi < p.N;
#pragma unroll
    for (int b = 0; b < NB; ++b) fw[b][lane] = in ? p.bound[b][xi] : 0.0;
    const double vmu = (MODE == MODE_UPD || MODE == MODE_RES) && in ? p.muk[xi] : 0.0;
    const double vph = (MODE == MODE_MARG || MODE == MODE_RES) && in ? p.phik[xi] : 0.0;
    __syncwarp();
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
                for (int b = 0; b < NB; ++b) f[b] = fw[b][q * Q + m];
                B *= wl;                   // edge (m, m+1)
                B = ls_place(B, f, mb);
            }
        }
    }
    // walk 2 (left to right): rebuild the Q suffix states of each block, prefix step, the terms
    // F[S] H[S^c] of the block's Q points, then one reduce-scatter of the Q sums over the lanes
    const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
    double tj = 0.0;  // J of this lane's point (lane j <-> x0 + j)
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
                for (int b = 0; b < NB; ++b) f[b] = fw[b][q * Q + i];
                st = ls_place(st, f, mb);
            }
        }
        double v[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            double f[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) f[b] = fw[b][q * Q + i];
            F *= wl;
            F = ls_place(F, f, mb);
            v[i] = F * __shfl_xor_sync(0xffffffffu, H[i], M - 1);  // F[S] H[S^c]
        }
        // reduce-scatter: after the three halving steps lane L holds the partial sum of point
        // q Q + (L >> 2) over its 4-lane group's share; two butterflies finish it
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double snd = b4 ? v[k] : v[k + 4], kp = b4 ? v[k + 4] : v[k];
            v[k] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double snd = b3 ? v[k] : v[k + 2], kp = b3 ? v[k + 2] : v[k];
            v[k] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
        }
        {
            const double snd = b2 ? v[0] : v[1], kp = b2 ? v[1] : v[0];
            v[0] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        const double x = __shfl_sync(0xffffffffu, v[0], 4 * (lane & 7));
        tj = (lane >> 3) == q ? x : tj;
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
    const size_t smb = 2 * kLsB * (size_t)kLsStride * sizeof(double);
    smem_attr((const void *)k_ls_blockscan<false>, smb);
    smem_attr((const void *)k_ls_blockscan<true>, smb);
    smem_attr((const void *)k_ls_prefix_red, smb);
    static const int tree0 = getenv("MMOT_LS_KS0") ? 0 : 1;  // level 0: tree (default) or Kogge-Stone
    static const int red_up = getenv("MMOT_LS_KS_UP") ? 0 : 1;  // upper levels: per-output trees
    // down pass: the top level inside its k_ls_prefix_red, level 1 inside k_ls_apply (no k_ls_down
    // launches for scans of <= 3 levels)
    static const int fuse_down = getenv("MMOT_LS_NO_FUSE_DOWN") ? 0 : 1;
    const bool top_fused = fuse_down && red_up && w.nlev >= 2;
    const int fuse1 = fuse_down && w.nlev >= 3 ? 1 : 0;
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
        L.car[0] = top_fused && lv == w.nlev - 1 ? w.lv_car[lv][0] : nullptr;
        L.car[1] = top_fused && lv == w.nlev - 1 ? w.lv_car[lv][1] : nullptr;
        const dim3 g((unsigned)((L.n + kLsB - 1) / kLsB), 2);
        if (lv == 0 && tree0) k_ls_blockscan<true><<<g, kLsB * 32, smb, s>>>(L, p.stop);
        else if (lv == 0 || !red_up) k_ls_blockscan<false><<<g, kLsB * 32, smb, s>>>(L, p.stop);
        else k_ls_prefix_red<<<dim3((unsigned)(L.n + (L.agg[0] ? g.x : 0)), 2), kLsB * 32, smb, s>>>(L, p.stop);
        ++nl;
    }
    // down: carries of every level from the top; level 0's are the chain carries (scan order)
    for (int lv = w.nlev - 1; lv >= 1; --lv) {  // level 0: inside k_ls_apply
        if ((top_fused && lv == w.nlev - 1) || (fuse1 && lv == 1)) continue;
        const int64_t n = w.lv_n[lv];
        const double *par0 = lv + 1 < w.nlev ? w.lv_car[lv + 1][0] : nullptr;
        const double *par1 = lv + 1 < w.nlev ? w.lv_car[lv + 1][1] : nullptr;
        k_ls_down<<<(unsigned)((2 * n + 3) / 4), 128, 0, s>>>(w.lv_excl[lv][0], w.lv_excl[lv][1], par0, par1,
                                                             w.lv_car[lv][0], w.lv_car[lv][1], n, p.stop);
        ++nl;
    }
    switch (mode) {
        case MODE_UPD: k_ls_apply<MODE_UPD><<<wb, 128, 0, s>>>(p, w, fuse1); break;
        case MODE_MARG: k_ls_apply<MODE_MARG><<<wb, 128, 0, s>>>(p, w, fuse1); break;
        default: k_ls_apply<MODE_RES><<<wb, 128, 0, s>>>(p, w, fuse1); break;
    }
    *launches += 2 + nl;
    return cudaGetLastError();
}

}  // namespace mmot
