// esa_deep.cu — Enumerate-Score-Argmax for deep patterns (k <= 16, N <= 32)
// on sm_100a (the paper's overhead study reaches
// "9 GPUs and above" on 16-GPU graphs).
//
// Why a second kernel: the narrow kernels (esa_kernels.cuh) put the devices
// of the LAST pattern vertex on the lanes and keep the DFS state of every
// level in registers, so (a) they need a packed 63-bit key (15 + W + C(k,2)
// bits: k <= 8 at W <= 16, k <= 6 at W = 32) and (b) when k approaches the
// free count only nF - k + 1 lanes per scan do work.  Here:
//   * vertices 0..T-1 (T = k - L) are placed by a warp-uniform DFS whose
//     stack is distributed over the lanes (lane j holds f(j), the candidates
//     left at level j and the partial score after j) and read back with
//     shuffles; the increment of placing vertex d on v is one table read per
//     lane j < d plus a warp reduction (REDUX), the lex-leader lower bound a
//     REDUX max;
//   * the last L vertices (L = 1..4, chosen on the host so a node has >= ~32
//     leaves) are a lane-parallel scan over a launch-constant table of
//     L-tuples of indices into the r = nF - T free devices left at every
//     node (sorted, so index order = device order and the suffix-internal
//     lex-leader constraints are applied once, on the host, when the table
//     is built).  Per node the lanes fill a partial table pt[l][i] (score of
//     suffix vertex T+l on the i-th remaining device w.r.t. the placed
//     prefix, by popc over class masks) and a pair table wt[i][i2]; a leaf is
//     then L + (#suffix-internal scored pairs) shared-memory reads and adds;
//   * the argmax key is 256 bits (score, brev64(S), 128-bit edge code),
//     compared lexicographically, so any k <= 16 fits on any N <= 64.  It is
//     built only for a leaf whose score reaches the lane's best.  CTAs merge
//     their best under a lock in the record (max is order independent:
//     deterministic for every grid size and rank count);
//   * device masks are a template type: u32 for N <= 32, u64 for N <= 64
//     (SURVEY §8(f) NEXT 4); only per-node work touches them.
// Scores are the narrow path's (integer): Eq. 1 AggBW, Eq. 2 as
// the dense rank of the census (host table, reading A9 holds for
// m <= 120), Eq. 3 PreservedBW = T_F - sum inc_F(S) + inside(S).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "internal.h"

namespace mapa {
namespace {

constexpr unsigned kFullD = 0xFFFFFFFFu;
constexpr int kBlockD = 256;
constexpr int kWarpsD = kBlockD / 32;
constexpr int kMaxDecodeD = 6;
constexpr int kMaxL = 4;
constexpr int kND = kMaxNDeep;
// per-warp term area (ints): pt[l][i] at l*64 + i, the pair table at
// kWtOff + i*kWtStride + i2 (odd stride: fewer bank conflicts), a zero at kZeroOff
constexpr int kWtOff = 256, kWtStride = 17, kZeroOff = 528, kAreaInts = 532;

struct DeepWarp {
    int area[kAreaInts];
    int dl[kND];     // remaining free devices, ascending
    int fw[16];      // f(j) of the placed prefix (read by the key builder)
};

// The tuple table (uint4 per tuple -- x: byte l = i_l; y, z, w: 16-bit byte
// offsets of the NT terms into area) follows the rank table, sized by ntup, so
// that small tables do not cost occupancy.
struct DeepShared {
    unsigned long long cm[kND][3];
    int tw[kND * kND];         // [v*64 + b] pair value: w(v,b) (Eq. 1/3), census delta (Eq. 2), 0 if v == b
    int incF[kND];             // inc_F(v) (Eq. 3)
    int maxw[kND];             // branch and bound: max_{u in F, u != v} w(u, v)
    int gmax;                  // branch and bound: max over free pairs
    uint32_t magic[kND + 4];
    DeepWarp w[kWarpsD];
    unsigned long long rk[kWarpsD][5];
};

// dynamic shared memory: DeepShared + the Eq. 2 rank table (u16, (m+1)^2 <= 121^2)
// [+ the Eq. 2 branch-and-bound tables, (k+1) (m+1)^2 <= kSensBoundMax u16]
// [+ the tuple table, ntup <= kMaxTup uint4]
constexpr int kDeepSmemMax =
    (int)sizeof(DeepShared) + 2 * (kMaxEdges + 1) * (kMaxEdges + 1) + 2 * kSensBoundMax + 16 + 16 * kMaxTup;
// byte offset of the tuple table: after DeepShared and the selector's rank (+ bound) tables
__host__ __device__ __forceinline__ int deep_tup_off(int sc, int xsd, int k) {
    const int lut = (sc & 3) == SEL_SENS ? 2 * xsd * xsd * (1 + ((sc & 8) ? k + 1 : 0)) : 0;
    return ((int)sizeof(DeepShared) + lut + 15) & ~15;
}

extern __shared__ __align__(16) unsigned char g_dsmem[];
__device__ __forceinline__ DeepShared &dsh() { return *reinterpret_cast<DeepShared *>(g_dsmem); }
__device__ __forceinline__ uint16_t *dlut() { return reinterpret_cast<uint16_t *>(g_dsmem + sizeof(DeepShared)); }
template <int SEL> __device__ __forceinline__ uint4 *dtup(const DeepTables &tb) {
    return reinterpret_cast<uint4 *>(g_dsmem + deep_tup_off(SEL, tb.xsd, tb.k));
}

// ---- mask helpers (M = uint32_t for N <= 32, unsigned long long for N <= 64)
template <typename M> __device__ __forceinline__ int popc(M m);
template <> __device__ __forceinline__ int popc<uint32_t>(uint32_t m) { return __popc(m); }
template <> __device__ __forceinline__ int popc<unsigned long long>(unsigned long long m) { return __popcll(m); }
template <typename M> __device__ __forceinline__ int lowbit(M m);
template <> __device__ __forceinline__ int lowbit<uint32_t>(uint32_t m) { return __ffs(m) - 1; }
template <> __device__ __forceinline__ int lowbit<unsigned long long>(unsigned long long m) { return __ffsll(m) - 1; }
template <typename M> __device__ __forceinline__ M bit(int d) { return M(1) << d; }
template <typename M> __device__ __forceinline__ M below(int d) { return (M(1) << d) - M(1); }  // d < width
// devices above d (d = -1: all)
template <typename M> __device__ __forceinline__ M above(int d) {
    constexpr int W = 8 * (int)sizeof(M);
    return d < 0 ? ~M(0) : (d + 1 >= W ? M(0) : (~M(0) << (d + 1)));
}
// devices up to and including d
template <typename M> __device__ __forceinline__ M upto(int d) {
    constexpr int W = 8 * (int)sizeof(M);
    return d + 1 >= W ? ~M(0) : ((M(1) << (d + 1)) - M(1));
}
template <typename M> __device__ __forceinline__ M reduce_or(M v);
template <> __device__ __forceinline__ uint32_t reduce_or<uint32_t>(uint32_t v) { return __reduce_or_sync(kFullD, v); }
template <> __device__ __forceinline__ unsigned long long reduce_or<unsigned long long>(unsigned long long v) {
    const uint32_t lo = __reduce_or_sync(kFullD, (uint32_t)v), hi = __reduce_or_sync(kFullD, (uint32_t)(v >> 32));
    return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ uint32_t nth_set32(uint32_t m, uint32_t n) {
    uint32_t pos = 0, c;
    c = __popc(m & 0xFFFFu); if (n >= c) { n -= c; m >>= 16; pos += 16; }
    c = __popc(m & 0xFFu);   if (n >= c) { n -= c; m >>= 8;  pos += 8; }
    c = __popc(m & 0xFu);    if (n >= c) { n -= c; m >>= 4;  pos += 4; }
    c = __popc(m & 0x3u);    if (n >= c) { n -= c; m >>= 2;  pos += 2; }
    c = m & 1u;              if (n >= c) { pos += 1; }
    return pos;
}
template <typename M> __device__ __forceinline__ uint32_t nth_set(M m, uint32_t n);
template <> __device__ __forceinline__ uint32_t nth_set<uint32_t>(uint32_t m, uint32_t n) { return nth_set32(m, n); }
template <> __device__ __forceinline__ uint32_t nth_set<unsigned long long>(unsigned long long m, uint32_t n) {
    const uint32_t lo = (uint32_t)m, c = (uint32_t)__popc(lo);
    return n < c ? nth_set32(lo, n) : 32u + nth_set32((uint32_t)(m >> 32), n - c);
}

struct DBest {
    uint32_t score;
    unsigned long long set;  // brev64(S); 0 = none
    unsigned long long ehi, elo;
};

__device__ __forceinline__ bool key_gt(uint32_t s0, unsigned long long a0, unsigned long long a1,
                                       unsigned long long a2, uint32_t s1, unsigned long long b0,
                                       unsigned long long b1, unsigned long long b2) {
    return s0 != s1 ? s0 > s1 : (a0 != b0 ? a0 > b0 : (a1 != b1 ? a1 > b1 : a2 > b2));
}

// A leaf whose (scaled) score reached the lane's threshold.  Builds the device
// set, and (unless the set alone decides) the 128-bit edge code: pattern edge
// (a, b) -> ranks ra, rb of f(a), f(b) inside S -> pair index p of (lo, hi)
// in lex order over C(k,2) -> bit C(k,2)-1-p.  Updates the lane's best key
// and threshold.
__device__ __forceinline__ void consider_deep(const DeepTables &tb, const DeepWarp &W, DBest &b, int &thr,
                                              uint32_t s, unsigned long long U, uint32_t x, int T,
                                              unsigned long long *gpub) {
    const int L = tb.L;
    unsigned long long S = U;
#pragma unroll
    for (int l = 0; l < kMaxL; ++l)
        if (l < L) S |= 1ull << W.dl[(x >> (8 * l)) & 0xFFu];
    const unsigned long long set = __brevll(S);
    if (s < b.score || (s == b.score && set < b.set)) return;
    if (s == b.score && set == b.set && tb.clique) return;  // same set of a clique: same edges
    const int k = tb.k, eb = tb.eb;
    unsigned long long ehi = 0, elo = 0;
    for (int e = 0; e < tb.m; ++e) {
        const int a = tb.edge[e] & 15, c = tb.edge[e] >> 4;
        const int da = a < T ? W.fw[a] : W.dl[(x >> (8 * (a - T))) & 0xFFu];
        const int dc = c < T ? W.fw[c] : W.dl[(x >> (8 * (c - T))) & 0xFFu];
        const int ra = __popcll(S & ((1ull << da) - 1ull)), rc = __popcll(S & ((1ull << dc) - 1ull));
        const int lo = min(ra, rc), hi2 = max(ra, rc);
        const int p = lo * (2 * k - lo - 1) / 2 + (hi2 - lo - 1);
        const int q = eb - 1 - p;
        if (q >= 64) ehi |= 1ull << (q - 64);
        else elo |= 1ull << q;
    }
    if (key_gt(s, set, ehi, elo, b.score, b.set, b.ehi, b.elo)) {
        if (gpub && (s > b.score || set > b.set))  // branch and bound: publish (score, top of brev64(S))
            atomicMax(gpub, ((unsigned long long)s << 32) | (set >> 32));
        b.score = s;
        b.set = set;
        b.ehi = ehi;
        b.elo = elo;
        thr = (int)s * tb.scale;
    }
}

// Increment of placing pattern vertex d on device v, given the lane-held
// prefix f(lane) for lane < d.  Eq. 1: back-neighbours of d; Eq. 3: every
// placed vertex, minus inc_F(v); Eq. 2: census delta; Baseline: 0.
template <int SEL>
__device__ __forceinline__ int place_inc(const DeepTables &tb, int d, int v, int myf, int lane) {
    constexpr int base = SEL & 3;
    if constexpr (base == SEL_BASE) return 0;
    int c = 0;
    const bool e = base == SEL_INSENS ? true : ((tb.back[d] >> lane) & 1u) != 0;
    if (lane < d && e) c = dsh().tw[myf * kND + v];
    int s = __reduce_add_sync(kFullD, c);
    if constexpr (base == SEL_INSENS) s -= dsh().incF[v];
    return s;
}

// Canonical mode: devices allowed for vertex d by its lex-leader sources.
template <typename M, int SEL>
__device__ __forceinline__ M allowed(const DeepTables &tb, int d, int myf, int lane) {
    if constexpr (!(SEL & 4)) return ~M(0);
    const int c = (lane < d && ((tb.src[d] >> lane) & 1u)) ? myf : -1;
    return above<M>(__reduce_max_sync(kFullD, c));
}

// Branch and bound: true when no leaf below a node (pattern vertices 0..nd-1
// placed on U, lane j < nd holding f(j), partial score a) can beat the best
// key published in the record's reserved word (score << 32 | brev64(S) >> 32).
// Eq. 1: every pattern edge from a placed vertex j to the unplaced part <= the
// best free link of f(j), every edge inside the unplaced part <= the best free
// pair.  Eq. 2: the largest rank reachable from the census so far (host table
// per nd).  On a score tie: the subtree's best set is U + the lowest k - nd
// other free devices; cut when even that set orders below the published one.
template <typename M, int SEL>
__device__ __forceinline__ bool bound_cut(const DeepTables &tb, M F, M U, int nd, int a, int myf, int lane,
                                          const unsigned long long *gpub) {
    constexpr int base = SEL & 3;
    const DeepShared &S = dsh();
    int ub;
    if constexpr (base == SEL_SENS) {
        ub = dlut()[tb.xsd * tb.xsd * (1 + nd) + a];
    } else {
        const int c = lane < nd ? __popc((uint32_t)tb.adj[lane] >> nd) * S.maxw[myf] : 0;
        ub = a + __reduce_add_sync(kFullD, c) + (int)tb.c2[nd] * S.gmax;
    }
    const unsigned long long gk = ld_relaxed(gpub);
    const unsigned gb = (unsigned)(gk >> 32);
    if (ub != (int)gb) return ub < (int)gb;
    const M R = F & ~U;
    const int need = tb.k - nd;
    const M low = need >= popc<M>(R) ? R : (R & below<M>((int)nth_set<M>(R, need)));
    return (uint32_t)(__brevll((unsigned long long)(U | low)) >> 32) < (uint32_t)gk;
}

// L = 2 without a tuple table (tb.lanes2; the host picks it when r is large,
// e.g. N = 64 topologies, where the 16x16 pair table of the tuple scan caps L
// at 1 and a node would hold only r leaves): vertex T walks the r remaining
// devices i (uniform loop, pt[0][i] and dl[i] broadcast from shared memory),
// vertex T+1 sits on the lanes j = lane, lane + 32 (pt[1][j] and dl[j] in
// registers); a leaf costs one gather of the pair value w(dl[i], dl[j]) from
// the 64x64 table, one add and the threshold test.  pt[l][i] is already in
// the area (scale 1: Eq. 3 is pt0 + pt1 + w, every pair scored).
template <typename M, int SEL>
__device__ __forceinline__ void suffix_lanes2(const DeepTables &tb, const DeepWarp &W, int r, int A, uint32_t MINI, M U,
                                              unsigned long long nbest, int lane, int T, DBest &bst, int &thr,
                                              unsigned long long &cnt, unsigned long long *gpub) {
    constexpr int base = SEL & 3;
    constexpr bool canon = (SEL & 4) != 0;
    constexpr bool prune = (SEL & 8) != 0;
    const DeepShared &S = dsh();
    const int mi0 = canon ? (int)(MINI & 0xFFu) : 0, mi1 = canon ? (int)((MINI >> 8) & 0xFFu) : 0;
    const bool dep = canon && tb.l2dep;
    const int e = tb.l2e;
    const int two = r > 32;
    __syncwarp();  // pt[l][i] and dl written by the other lanes
    int pj0 = 0, pj1 = 0, dj0 = 0, dj1 = 0;
    if (lane < r) { pj0 = W.area[kND + lane]; dj0 = W.dl[lane]; }
    if (two && lane + 32 < r) { pj1 = W.area[kND + lane + 32]; dj1 = W.dl[lane + 32]; }
    // leaves of this node (closed form): i in [mi0, r), j in [mi1, r), j != i (dep: j > i)
    {
        int c = 0;
        for (int i = mi0 + lane; i < r; i += 32) c += r - max(mi1, dep ? i + 1 : 0) - (!dep && i >= mi1 ? 1 : 0);
        cnt += (unsigned long long)__reduce_add_sync(kFullD, c);
    }
    if constexpr (prune && base != SEL_SENS) {
        // every leaf <= A + max pt0 + max pt1 + e * (best free pair)
        int m0 = kNegTable, m1 = kNegTable;
        if (lane >= mi0 && lane < r) m0 = W.area[lane];
        if (lane + 32 >= mi0 && lane + 32 < r) m0 = max(m0, W.area[lane + 32]);
        if (lane >= mi1 && lane < r) m1 = pj0;
        if (lane + 32 >= mi1 && lane + 32 < r) m1 = max(m1, pj1);
        const int ub = A + __reduce_max_sync(kFullD, m0) + __reduce_max_sync(kFullD, m1) + e * S.gmax;
        const unsigned gb = (unsigned)(ld_relaxed(gpub) >> 32);
        if (ub < (int)gb) return;
    }
    int tie = nbest >= bst.set ? 0 : 1;  // score ties (see suffix)
    for (int i = mi0; i < r; ++i) {
        const int a = A + W.area[i];
        const int *row = S.tw + W.dl[i] * kND;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h == 1 && !two) break;
            const int j = lane + 32 * h;
            const bool valid = j < r && j >= mi1 && (dep ? j > i : j != i);
            int s = a + (h ? pj1 : pj0) + (e ? row[h ? dj1 : dj0] : 0);
            if constexpr (base == SEL_SENS) s = dlut()[valid ? s : 0];
            if (valid && s >= thr + tie) {
                consider_deep(tb, W, bst, thr, (uint32_t)s, (unsigned long long)U, (uint32_t)i | ((uint32_t)j << 8), T,
                              prune ? gpub : nullptr);
                tie = nbest >= bst.set ? 0 : 1;
            }
        }
    }
    __syncwarp();
}

// All leaves below a node whose prefix 0..T-1 is placed (set U, score A).
template <typename M, int NT, int SEL>
__device__ __forceinline__ void suffix(const DeepTables &tb, M F, M U, int A, int myf, int lane, int warp, int T,
                                       DBest &bst, int &thr, unsigned long long &cnt, unsigned long long *gpub) {
    constexpr int base = SEL & 3;
    constexpr bool canon = (SEL & 4) != 0;
    constexpr bool prune = (SEL & 8) != 0;
    DeepShared &S = dsh();
    DeepWarp &W = S.w[warp];
    const int L = tb.L;
    M R = F & ~U;
    if constexpr (canon) {
        // lower bound shared by every suffix vertex: drop the devices below it
        if (tb.pcommon) R &= above<M>(__reduce_max_sync(kFullD, (lane < T && ((tb.pcommon >> lane) & 1)) ? myf : -1));
    }
    const int r = popc<M>(R);
    // Score ties: a leaf of this node holds U plus L devices of R, so the best
    // device set any of them can have is U + the L lowest devices of R.  When
    // that set orders below the lane's best set, a leaf that only TIES the
    // lane's best score cannot win the tie-break: the threshold is strict
    // (scores are multiples of `scale`), and such leaves -- every automorphic
    // copy of a winner in RAW mode, and equal-weight labellings on topologies
    // with many equal links -- never reach the out-of-line key builder.
    const M lowL = L >= r ? R : (R & below<M>((int)nth_set<M>(R, (uint32_t)L)));
    const unsigned long long nbest = __brevll((unsigned long long)(U | lowL));
    __syncwarp();  // previous readers of dl / area are done
#pragma unroll
    for (int h = 0; h < (int)sizeof(M) / 4; ++h) {
        const int dv = lane + 32 * h;
        if ((R >> dv) & 1u) W.dl[popc<M>(R & below<M>(dv))] = dv;
    }
    M X[kMaxL];
    uint32_t MINI = 0;
#pragma unroll
    for (int l = 0; l < kMaxL; ++l) {
        X[l] = 0;
        if (l < L) {
            const int u = T + l;
            if constexpr (base == SEL_INSENS) X[l] = U;
            else X[l] = reduce_or<M>((lane < T && ((tb.back[u] >> lane) & 1u)) ? bit<M>(myf) : M(0));
            if constexpr (canon) {
                if (tb.pcon) {
                    const int lb = __reduce_max_sync(kFullD, (lane < T && ((tb.src[u] & ~tb.pcommon) >> lane) & 1u) ? myf : -1);
                    const uint32_t mi = lb < 0 ? 0u : (uint32_t)popc<M>(R & upto<M>(lb));
                    MINI |= mi << (8 * l);
                }
            }
        }
    }
    __syncwarp();
    for (int i = lane; i < r; i += 32) {
        const int dev = W.dl[i];
        const M c0 = (M)S.cm[dev][0], c1 = (M)S.cm[dev][1], c2 = (M)S.cm[dev][2];
#pragma unroll
        for (int l = 0; l < kMaxL; ++l) {
            if (l < L) {
                int v;
                if constexpr (base == SEL_SENS) {
                    v = popc<M>(c0 & X[l]) * tb.xsd + popc<M>((c1 | c2) & X[l]);
                } else if constexpr (base == SEL_BASE) {
                    v = 0;
                } else {
                    v = 12 * popc<M>(X[l]) + 38 * popc<M>(c0 & X[l]) + 13 * popc<M>(c1 & X[l]) + 8 * popc<M>(c2 & X[l]);
                    if constexpr (base == SEL_INSENS) v -= S.incF[dev];
                }
                W.area[kND * l + i] = v;
            }
        }
    }
    if (tb.lanes2) {
        suffix_lanes2<M, SEL>(tb, W, r, A, MINI, U, nbest, lane, T, bst, thr, cnt, gpub);
        return;
    }
    // Pair table.  Eq. 3 with L >= 2 (scale = L-1): the score depends on the
    // set only and pt[l][i] = q[i] for every l, so
    //   (L-1) s = (L-1) A + sum over the C(L,2) pairs of (L-1) w(i, i2) + q[i] + q[i2]
    // and the tuple terms are the pairs alone.
    if (tb.nes) {
        __syncwarp();  // pt written
        const int sc = tb.scale;
        const bool fold = base == SEL_INSENS && L >= 2;
        for (int p = lane; p < r * 16; p += 32) {
            const int i = p >> 4, i2 = p & 15;
            if (i2 < r) {
                int v = S.tw[W.dl[i] * kND + W.dl[i2]];
                if (fold) v = sc * v + W.area[i] + W.area[i2];
                W.area[kWtOff + i * kWtStride + i2] = v;
            }
        }
    }
    __syncwarp();
    const int nt = tb.tcount[r];
    const char *ab = reinterpret_cast<const char *>(W.area);
    const int A0 = A * tb.scale;
    if constexpr (prune && base != SEL_SENS) {
        // table bound: every tuple's score <= A + sum over its terms of the
        // largest entry its table can hold; strict test against the grid best
        int ub = A0;
        for (int q = 0; q < tb.nterm; ++q) {
            int mx = kNegTable;
            if (tb.term[q][0] == 0) {
                for (int i = lane; i < r; i += 32) mx = max(mx, W.area[kND * tb.term[q][1] + i]);
            } else {
                for (int p = lane; p < r * 16; p += 32)
                    if ((p & 15) < r) mx = max(mx, W.area[kWtOff + (p >> 4) * kWtStride + (p & 15)]);
            }
            ub += __reduce_max_sync(kFullD, mx);
        }
        const unsigned gb = (unsigned)(ld_relaxed(gpub) >> 32);
        if (ub < (int)gb * tb.scale) {  // scaled units (Eq. 3 pair folding)
            __syncwarp();
            return;  // no tuple of this node can reach the best score found anywhere
        }
    }
    int tie = nbest >= bst.set ? 0 : 1;
    const uint4 *tupl = dtup<SEL>(tb);
    for (int t0 = 0; t0 < nt; t0 += 32) {
        const int t = t0 + lane;
        bool valid = t < nt;
        const uint4 e = tupl[valid ? t : 0];
        if constexpr (canon) {
            if (tb.pcon) valid = valid && ((((e.x | 0x80808080u) - MINI) & 0x80808080u) == 0x80808080u);
        }
        int s = A0;
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            const uint32_t wd = q < 2 ? e.y : (q < 4 ? e.z : e.w);
            const uint32_t off = (q & 1) ? (wd >> 16) : (wd & 0xFFFFu);
            s += *reinterpret_cast<const int *>(ab + off);
        }
        if constexpr (base == SEL_SENS) s = dlut()[s];
        if constexpr (canon) {
            if (tb.pcon) cnt += (unsigned long long)__popc(__ballot_sync(kFullD, valid));
        }
        if (valid && s >= thr + tie) {
            const int sc = tb.scale;
            const uint32_t sr = sc == 1 ? (uint32_t)s : (sc == 2 ? (uint32_t)s >> 1 : (uint32_t)s / 3u);
            consider_deep(tb, W, bst, thr, sr, (unsigned long long)U, e.x, T, prune ? gpub : nullptr);
            tie = nbest >= bst.set ? 0 : 1;
        }
    }
    if (!canon || !tb.pcon) cnt += (unsigned long long)nt;
    __syncwarp();  // lanes still reading fw / dl in consider_deep are done before the next push writes them
}

__device__ __forceinline__ uint32_t perm_count_d(int n, int d) {
    uint32_t p = 1;
    for (int j = 0; j < d; ++j) p *= (uint32_t)(n - j);
    return p;
}

template <typename M, int NT, int SEL>
__global__ void __launch_bounds__(kBlockD, 4)  // 64 registers (no spills), 4 CTAs per SM
esa_deep(const __grid_constant__ DeepTables tb, const uint16_t *__restrict__ lut_g,
         const mapa_query64 *__restrict__ dq, mapa_wide_record *__restrict__ rec, int D, int rank, int world,
         int stripe) {
    constexpr int base = SEL & 3;
    constexpr bool canon = (SEL & 4) != 0;
    DeepShared &S = dsh();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = tb.n;
    const M F = (M)(~dq->busy) & (n >= 8 * (int)sizeof(M) ? ~M(0) : below<M>(n));
    const int nF = popc<M>(F);
    const int T = tb.T;
    if (tid < kND) {
        S.cm[tid][0] = tb.cm[tid][0];
        S.cm[tid][1] = tb.cm[tid][1];
        S.cm[tid][2] = tb.cm[tid][2];
    }
    if (tid <= kND) S.magic[tid] = tid >= 2 ? (0xFFFFFFFFu / (uint32_t)tid + 1u) : 0u;
    if (lane == 0) S.w[warp].area[kZeroOff] = 0;
    for (int i = tid; i < kND * kND; i += kBlockD) {
        const int v = i / kND, b = i % kND;
        int val = 0;
        if (v != b && v < n && b < n) {
            const int cls = ((tb.cm[b][0] >> v) & 1u) ? 0 : ((tb.cm[b][1] >> v) & 1u) ? 1 : ((tb.cm[b][2] >> v) & 1u) ? 2 : 3;
            if constexpr (base == SEL_SENS) val = cls == 0 ? tb.xsd : (cls == 3 ? 0 : 1);
            else val = cls == 0 ? 50 : (cls == 1 ? 25 : (cls == 2 ? 20 : 12));  // Table 1
        }
        S.tw[i] = val;
    }
    // tuple entries: the term offsets of every tuple (pt[a][i_a] or the pair (i_a, i_b))
    for (int i = tid; i < tb.ntup; i += kBlockD) {
        const uint32_t x = tb.tup[i];
        uint32_t wd[3] = {kZeroOff * 4u * 0x10001u, kZeroOff * 4u * 0x10001u, kZeroOff * 4u * 0x10001u};
        for (int q = 0; q < tb.nterm; ++q) {
            const int a = tb.term[q][1], b = tb.term[q][2];
            const uint32_t ia = (x >> (8 * a)) & 0xFFu, ib = (x >> (8 * b)) & 0xFFu;
            const uint32_t off = 4u * (tb.term[q][0] == 0 ? (uint32_t)(kND * a) + ia : kWtOff + ia * kWtStride + ib);
            const int sh = 16 * (q & 1);
            wd[q >> 1] = (wd[q >> 1] & ~(0xFFFFu << sh)) | (off << sh);
        }
        dtup<SEL>(tb)[i] = make_uint4(x, wd[0], wd[1], wd[2]);
    }
    if constexpr (base == SEL_SENS) {
        const int nl = tb.xsd * tb.xsd * (1 + ((SEL & 8) ? tb.k + 1 : 0));  // + bound tables (prune)
        for (int i = tid; i < nl; i += kBlockD) dlut()[i] = lut_g[i];
    }
    if (tid < kND) {
        int inc = 0;
        if (tid < n && ((F >> tid) & 1u))
            inc = 12 * (nF - 1) + 38 * popc<M>((M)tb.cm[tid][0] & F) + 13 * popc<M>((M)tb.cm[tid][1] & F) +
                  8 * popc<M>((M)tb.cm[tid][2] & F);
        S.incF[tid] = inc;
    }
    constexpr bool prune = (SEL & 8) != 0;
    if (tid == 0 && nF != tb.r + T && tb.k <= nF) atomicOr(&rec->status, 2u);  // busy_hint mismatch
    __syncthreads();
    if constexpr (prune) {  // per-device best free link and the best free pair (tw is complete now)
        if (tid < kND) {
            int mw = 0;
            if (tid < n && ((F >> tid) & 1u))
                for (int u = 0; u < n; ++u)
                    if (u != tid && ((F >> u) & 1u)) mw = max(mw, S.tw[u * kND + tid]);
            S.maxw[tid] = mw;
        }
        __syncthreads();
        if (warp == 0) {
            const int g2 = __reduce_max_sync(kFullD, max(S.maxw[lane], S.maxw[lane + 32]));
            if (lane == 0) S.gmax = g2;
        }
        __syncthreads();
    }
    unsigned long long *gpub = prune ? reinterpret_cast<unsigned long long *>(&rec->reserved) : nullptr;
    int acc0 = 0;
    if constexpr (base == SEL_INSENS) acc0 = __reduce_add_sync(kFullD, S.incF[lane] + S.incF[lane + 32]) / 2;  // T_F

    // Rank-local item space and guided self-scheduling, as the narrow kernel.
    const bool okq = tb.k <= nF && nF == tb.r + T;
    const uint32_t N = okq ? perm_count_d(nF, D) : 0u;
    const uint32_t Ls = (uint32_t)stripe;
    const uint32_t nS = (N + Ls - 1u) / Ls;
    const uint32_t myS = nS > (uint32_t)rank ? (nS - (uint32_t)rank + (uint32_t)world - 1u) / (uint32_t)world : 0u;
    const bool ownLast = nS > 0 && ((nS - 1u) % (uint32_t)world) == (uint32_t)rank;
    const uint32_t Nloc = myS == 0 ? 0u : (ownLast ? (myS - 1u) * Ls + (N - (nS - 1u) * Ls) : myS * Ls);
    const uint32_t P = gridDim.x * (uint32_t)kWarpsD;
    DBest bst{0u, 0ull, 0ull, 0ull};
    int thr = 0;
    unsigned long long cnt = 0;
    int myf = 0, myacc = 0;
    M mycand = 0;
    for (;;) {
        uint32_t start = 0, sz = 0;
        if (lane == 0) {
            const uint32_t cur = ld_relaxed(&rec->ctr);
            const uint32_t rem = cur < Nloc ? Nloc - cur : 0u;
            sz = max(1u, rem / (2u * P));
            start = atomicAdd(&rec->ctr, sz);
        }
        start = __shfl_sync(kFullD, start, 0);
        sz = __shfl_sync(kFullD, sz, 0);
        if (start >= Nloc) break;
        const uint32_t end = min(start + sz, Nloc);
        for (uint32_t j = start; j < end; ++j) {
            const uint32_t sl = j / Ls;
            uint32_t item = (sl * (uint32_t)world + (uint32_t)rank) * Ls + (j - sl * Ls);
            // decode the prefix of depth D (mixed radix nF - q at level q).
            // Level 0 is the LEAST significant digit: under lex-leader bounds
            // the prefixes with a small f(0) are far heavier, and this order
            // interleaves them with light ones so that every chunk of
            // consecutive items carries about the average work.
            uint32_t dg[kMaxDecodeD];
#pragma unroll
            for (int q = 0; q < kMaxDecodeD; ++q) {
                if (q < D) {
                    const uint32_t rr = (uint32_t)(nF - q);
                    const uint32_t qq = __umulhi(item, S.magic[rr]);
                    dg[q] = item - qq * rr;
                    item = qq;
                } else {
                    dg[q] = 0;
                }
            }
            M U = 0;
            int acc = acc0;
            bool ok = true;
#pragma unroll
            for (int q = 0; q < kMaxDecodeD; ++q) {
                if (q < D) {
                    const int v = (int)nth_set<M>(F & ~U, dg[q]);
                    if (canon && !((allowed<M, SEL>(tb, q, myf, lane) >> v) & 1u)) { ok = false; break; }
                    acc += place_inc<SEL>(tb, q, v, myf, lane);
                    if (lane == q) { myf = v; myacc = acc; }
                    if (lane == 0) S.w[warp].fw[q] = v;
                    U |= bit<M>(v);
                }
            }
            if (!ok) continue;
            if constexpr (prune)  // the item's own subtree (prefix 0..D-1 placed)
                if (D > 0 && bound_cut<M, SEL>(tb, F, U, D, acc, myf, lane, gpub)) continue;
            if (D == T) {
                suffix<M, NT, SEL>(tb, F, U, acc, myf, lane, warp, T, bst, thr, cnt, gpub);
                continue;
            }
            // explicit-stack DFS over levels D..T-1 (lane d holds level d)
            int d = D;
            M cand = F & ~U & allowed<M, SEL>(tb, d, myf, lane);
            for (;;) {
                if (cand == 0) {
                    if (d == D) break;
                    --d;
                    const int v = __shfl_sync(kFullD, myf, d);
                    U &= ~bit<M>(v);
                    cand = __shfl_sync(kFullD, mycand, d);
                    continue;
                }
                const int v = lowbit<M>(cand);
                cand &= cand - M(1);
                const int accp = d == 0 ? acc0 : __shfl_sync(kFullD, myacc, d - 1);
                const int a = accp + place_inc<SEL>(tb, d, v, myf, lane);
                if (lane == d) { myf = v; mycand = cand; myacc = a; }
                if (lane == 0) S.w[warp].fw[d] = v;
                U |= bit<M>(v);
                if constexpr (prune) {
                    if (bound_cut<M, SEL>(tb, F, U, d + 1, a, myf, lane, gpub)) {
                        U &= ~bit<M>(v);
                        continue;  // skip the subtree: try the next candidate of level d
                    }
                }
                if (d + 1 == T) {
                    suffix<M, NT, SEL>(tb, F, U, a, myf, lane, warp, T, bst, thr, cnt, gpub);
                    U &= ~bit<M>(v);
                } else {
                    ++d;
                    cand = F & ~U & allowed<M, SEL>(tb, d, myf, lane);
                }
            }
        }
    }
    // warp / block / grid lexicographic max of the 256-bit key
    uint32_t hs = bst.score;
    unsigned long long h = bst.set, e1 = bst.ehi, e0 = bst.elo;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t s2 = __shfl_xor_sync(kFullD, hs, o);
        const unsigned long long h2 = __shfl_xor_sync(kFullD, h, o);
        const unsigned long long a2 = __shfl_xor_sync(kFullD, e1, o);
        const unsigned long long b2 = __shfl_xor_sync(kFullD, e0, o);
        if (key_gt(s2, h2, a2, b2, hs, h, e1, e0)) { hs = s2; h = h2; e1 = a2; e0 = b2; }
    }
    if (lane == 0) {
        S.rk[warp][0] = hs;
        S.rk[warp][1] = h;
        S.rk[warp][2] = e1;
        S.rk[warp][3] = e0;
        S.rk[warp][4] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long c = 0;
        hs = 0; h = 0; e1 = 0; e0 = 0;
        for (int w = 0; w < kWarpsD; ++w) {
            c += S.rk[w][4];
            if (key_gt((uint32_t)S.rk[w][0], S.rk[w][1], S.rk[w][2], S.rk[w][3], hs, h, e1, e0)) {
                hs = (uint32_t)S.rk[w][0]; h = S.rk[w][1]; e1 = S.rk[w][2]; e0 = S.rk[w][3];
            }
        }
        if (c) atomicAdd(reinterpret_cast<unsigned long long *>(&rec->leaves), c);
        // Filter before the lock: (score, top 32 bits of the set word) orders
        // keys consistently with the full 256-bit order, so a CTA whose packed
        // value is below the running maximum cannot win and skips the
        // serialised merge (without it every CTA took the lock: ~640 us per
        // launch at 444 CTAs).
        const unsigned long long packed = ((unsigned long long)hs << 32) | (h >> 32);
        if (h && atomicMax(reinterpret_cast<unsigned long long *>(&rec->reserved), packed) <= packed) {
            while (atomicCAS(&rec->lock, 0u, 1u) != 0u) {
            }
            __threadfence();
            volatile unsigned long long *r = reinterpret_cast<volatile unsigned long long *>(rec);
            if (r[1] == 0 || key_gt(hs, h, e1, e0, (uint32_t)r[0], r[1], r[2], r[3])) {
                r[0] = hs;
                r[1] = h;
                r[2] = e1;
                r[3] = e0;
            }
            __threadfence();
            atomicExch(&rec->lock, 0u);
        }
    }
}

template <typename M, int NT, int SEL>
int launch_t(const DeepTables &tb, const uint16_t *lut, const mapa_query64 *dq, mapa_wide_record *rec, int D,
             int rank, int world, int stripe, int grid, int smem, cudaStream_t st) {
    // the attribute is always the fixed upper bound, so occupancy queries and
    // launches agree
    // kernel attributes are per device: one flag bit per device ordinal
    static std::atomic<unsigned long long> configured{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return (int)cudaErrorInvalidDevice;
    if (!((configured.load(std::memory_order_relaxed) >> dev) & 1ull)) {
        cudaError_t e = cudaFuncSetAttribute((const void *)esa_deep<M, NT, SEL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kDeepSmemMax);
        if (e != cudaSuccess) return (int)e;
        configured.fetch_or(1ull << dev);
    }
    if (smem > kDeepSmemMax) return (int)cudaErrorInvalidValue;
    esa_deep<M, NT, SEL><<<grid, kBlockD, smem, st>>>(tb, lut, dq, rec, D, rank, world, stripe);
    return (int)cudaGetLastError();
}

using DeepFn = int (*)(const DeepTables &, const uint16_t *, const mapa_query64 *, mapa_wide_record *, int, int,
                       int, int, int, int, cudaStream_t);

template <typename M, int NT>
DeepFn pick_sel(int sc) {
    switch (sc & 15) {  // branch and bound: Greedy (8, 12), Preserve-sensitive (10, 14)
        case 8: return launch_t<M, NT, 8>;
        case 12: return launch_t<M, NT, 12>;
        case 10: return launch_t<M, NT, 10>;
        case 14: return launch_t<M, NT, 14>;
    }
    switch (sc & 7) {
        case 0: return launch_t<M, NT, 0>;
        case 1: return launch_t<M, NT, 1>;
        case 2: return launch_t<M, NT, 2>;
        case 3: return launch_t<M, NT, 3>;
        case 4: return launch_t<M, NT, 4>;
        case 5: return launch_t<M, NT, 5>;
        case 6: return launch_t<M, NT, 6>;
        default: return launch_t<M, NT, 7>;
    }
}

template <typename M, int NT>
const void *pick_fn_sel(int sc) {
    switch (sc & 15) {
        case 8: return (const void *)esa_deep<M, NT, 8>;
        case 12: return (const void *)esa_deep<M, NT, 12>;
        case 10: return (const void *)esa_deep<M, NT, 10>;
        case 14: return (const void *)esa_deep<M, NT, 14>;
    }
    switch (sc & 7) {
        case 0: return (const void *)esa_deep<M, NT, 0>;
        case 1: return (const void *)esa_deep<M, NT, 1>;
        case 2: return (const void *)esa_deep<M, NT, 2>;
        case 3: return (const void *)esa_deep<M, NT, 3>;
        case 4: return (const void *)esa_deep<M, NT, 4>;
        case 5: return (const void *)esa_deep<M, NT, 5>;
        case 6: return (const void *)esa_deep<M, NT, 6>;
        default: return (const void *)esa_deep<M, NT, 7>;
    }
}

// compile-time term count: the smallest of {2, 4, 6} >= nterm (padding terms read a zero)
inline int nt_class(int nterm) { return nterm <= 2 ? 2 : (nterm <= 4 ? 4 : 6); }

template <typename M>
DeepFn pick(int nterm, int sc) {
    switch (nt_class(nterm)) {
        case 2: return pick_sel<M, 2>(sc);
        case 4: return pick_sel<M, 4>(sc);
        default: return pick_sel<M, 6>(sc);
    }
}

template <typename M>
const void *pick_fn(int nterm, int sc) {
    switch (nt_class(nterm)) {
        case 2: return pick_fn_sel<M, 2>(sc);
        case 4: return pick_fn_sel<M, 4>(sc);
        default: return pick_fn_sel<M, 6>(sc);
    }
}

}  // namespace

int launch_deep(const DeepTables &tb, int sc, const uint16_t *d_lut, const mapa_query64 *d_query,
                mapa_wide_record *d_record, int depth, int rank, int world, int stripe, int grid, void *stream) {
    if (tb.ntup < 0 || tb.ntup > kMaxTup) return (int)cudaErrorInvalidValue;
    const int smem = deep_tup_off(sc, tb.xsd, tb.k) + 16 * tb.ntup;
    if (tb.nterm > kDeepMaxTerms || tb.L < 1 || tb.L > kMaxL) return (int)cudaErrorInvalidValue;
    DeepFn f = tb.n <= 32 ? pick<uint32_t>(tb.nterm, sc) : pick<unsigned long long>(tb.nterm, sc);
    return f(tb, d_lut, d_query, d_record, depth, rank, world, stripe, grid, smem, (cudaStream_t)stream);
}

int max_blocks_per_sm_deep(int n, int nterm, int sc, int lut_bytes) {
    // cached per (mask width, term class, selector code, rank-table size)
    static int cache[2][3][16][26] = {};
    const int mi = n <= 32 ? 0 : 1, ti = nt_class(nterm) / 2 - 1, li = std::min(25, (lut_bytes + 4095) / 4096);
    int &slot = cache[mi][ti][sc & 15][li];
    if (slot) return slot;
    const void *f = n <= 32 ? pick_fn<uint32_t>(nterm, sc) : pick_fn<unsigned long long>(nterm, sc);
    const int smem = (int)sizeof(DeepShared) + li * 4096;  // the bucket's upper bound
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kDeepSmemMax) != cudaSuccess) return 1;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kBlockD, smem) != cudaSuccess) return 1;
    slot = nb > 0 ? nb : 1;
    return slot;
}

}  // namespace mapa
