// esa.cu — Enumerate-Score-Argmax kernels for sm_100a (B200).
//
// One pass = SURVEY.md §8(a) S3-S6 fused in registers / shared memory:
//   S3 occupancy prep   F = ~busy; inc_F(v), T_F (Eq. 3 support)
//   S4 enumeration      DFS over injective maps f: V(P) -> F (§3.3 P:496-501;
//                       G complete, so every injective map embeds).
//                       Lanes = devices of the LAST pattern vertex k-1; the
//                       inner loop walks the devices v of vertex k-2.  Groups
//                       of W lanes (W = 8/16/32 = padded N) each run their own
//                       prefix, so small topologies still fill the warp.
//                       Canonical mode adds lex-leader lower bounds (one leaf
//                       per Aut(P)-orbit = SPEC dedup S:209).
//   S5 scoring          integer only.  With v's class masks c0..c2 and any
//                       device set X not containing v:
//                         sum_{u in X} w(u,v) = 12|X| + 38 popc(c0&X)
//                                               + 13 popc(c1&X) + 8 popc(c2&X)
//                       Outer DFS levels use that (popc, lane-uniform); the
//                       inner loop uses no popc at all: per prefix the lanes
//                       precompute in parallel (a) the score increment of
//                       placing vertex k-2 on their device (broadcast through
//                       a 32-entry smem list) and (b) their own leaf partial
//                       over vertices 0..k-3; each inner iteration then adds
//                       one list entry and one 32x32 weight-table byte.
//                         Eq. 1 AggBW: X = back-neighbour devices.
//                         Eq. 3 PreservedBW: T_F - sum inc_F(S)
//                         + inside(S), X = all placed devices.
//                         Eq. 2: census (x, y) accumulated as a
//                         table index x*(m+1)+y; score = dense rank of Eq. 2
//                         among the censuses with x+y+z = m (host table).
//   S6 argmax           per-lane running max of a packed 64-bit key (score |
//                       brev(S) | edge code), built out of line only when the
//                       score reaches the lane's best; warp shuffle max, block
//                       max, atomicMax in HBM.  Max is order independent, so
//                       the result is identical for every grid / rank count.
// Work items: the prefixes of depth D (mixed radix over the free devices),
// handed out as contiguous chunks; a chunk is walked as a DFS range, so only
// the first item of a run is decoded.  No dense contraction exists, so no
// tensor cores are used; the bound is integer issue.
#include <cuda_runtime.h>

#include "internal.h"

namespace mapa {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kMaxDecode = 4;

enum { SEL_LIN = 0, SEL_SENS = 1 };

struct Ctx {
    uint32_t F;
    int nF;
    int b;                          // lane's device id (lane % W)
    uint32_t gmask;                 // lanes of this lane's group
    uint32_t cm0, cm1, cm2, cm12;   // lane's class masks
    int incb;                       // inc_F(b)
    int laneC;                      // lane constant of the score (Eq. 3: -inc_F(b))
    int leafC;                      // k = 1 leaf constant
    int w0, w1, w2, w12;            // 38, 13, 8, 12 (0 for Baseline)
    int useU;                       // 1: X = all placed devices (Eq. 3), 0: back neighbours
    int acc0;                       // accumulator at the root (T_F for Eq. 3)
    const uint4 *cm;                // class masks of every device (smem)
    const int *inc;                 // inc_F(v) (smem)
    const uint16_t *lut;            // Eq. 2 table: (rank + 1) * 32 at [x * xs + y] (smem)
    const int *tw, *tz, *twd, *tzd; // inner-loop tables [v*32 + b] (smem, see SmemTopo)
    const int *tdl;                 // census index delta of edge (v, b) (smem)
    int4 *list;                     // this group's inner-loop candidate list (smem, W entries)
    int xs;                         // row stride of the Eq. 2 table (16 or 32)
    int mp1;                        // m + 1
    uint64_t fb, fs, db;            // bytes: fwd_back, fwd_src, dback
    int clique, eb, m;
    const uint8_t *edge;            // pattern edges a | b<<4
};

template <int K>
struct St {
    uint32_t U;       // placed devices
    int acc;          // LIN: partial score; SENS: x
    int acc2;         // SENS: y
    uint32_t f[K];    // f(i) for placed vertices
    uint32_t bm[K];   // bm[u]: devices of the placed back-neighbours of u
    uint32_t al[K];   // al[u]: devices allowed for u by lex-leader constraints
};

struct Best {
    unsigned long long key;
    uint32_t bs;
    uint32_t cnt;
};

// Inner-loop leaves are ranked by one int: (score + 1) * 32 + (31 - v).  Its
// max is the max score with ties to the smallest v.  Invalid leaves (vertex
// K-1 on the device of K-2, or a lex-leader violation) get kNeg added.
constexpr int kNeg = -(1 << 28);

// Per-CTA topology tables (shared memory), all indexed [v * 32 + b]:
//   tw  = 32 * w(v,b), kNeg when v == b or either is not a device
//   tz  = 0,           kNeg likewise
//   twd / tzd = the same with kNeg also where v >= b (canonical f(K-2) < f(K-1))
//   tdl = census index delta of the edge (v,b): xs * [double] + [single]
struct SmemTopo {
    uint4 cm[kMaxN];
    uint32_t magic[kMaxN + 1];
    int tw[kMaxN * kMaxN], tz[kMaxN * kMaxN], twd[kMaxN * kMaxN], tzd[kMaxN * kMaxN];
    int tdl[kMaxN * kMaxN];
};

__device__ __forceinline__ unsigned long long *u64p(uint64_t *p) {
    return reinterpret_cast<unsigned long long *>(p);
}

__device__ __forceinline__ uint32_t nth_set(uint32_t m, uint32_t n) {
    // position of the n-th (0-based) set bit of m (popc binary search)
    uint32_t pos = 0, c;
    c = __popc(m & 0xFFFFu); if (n >= c) { n -= c; m >>= 16; pos += 16; }
    c = __popc(m & 0xFFu);   if (n >= c) { n -= c; m >>= 8;  pos += 8; }
    c = __popc(m & 0xFu);    if (n >= c) { n -= c; m >>= 4;  pos += 4; }
    c = __popc(m & 0x3u);    if (n >= c) { n -= c; m >>= 2;  pos += 2; }
    c = m & 1u;              if (n >= c) { pos += 1; }
    return pos;
}

// Packed argmax key: score | brev_W(S) | edge code.  Only
// evaluated on the slow path (score >= the lane's best score), so it is kept
// out of line; arguments by value so the DFS state stays in registers.
//   fpack: f(0..K-2) one byte each; b: device of vertex K-1.
template <int W, int K>
__device__ __noinline__ unsigned long long make_key(uint32_t S, unsigned long long fpack, uint32_t b,
                                                    uint32_t s, int clique, int eb, int m,
                                                    const uint8_t *edge) {
    const uint32_t sb = __brev(S) >> (32 - W);
    uint32_t ecode;
    if (clique) {
        ecode = (1u << eb) - 1u;  // eb <= 28
    } else {
        uint32_t R = 0;  // rank of f(i) inside S, 4 bits per pattern vertex
#pragma unroll
        for (int i = 0; i < K - 1; ++i) {
            const uint32_t fi = (uint32_t)(fpack >> (8 * i)) & 0xFFu;
            R |= (uint32_t)__popc(S & ((1u << fi) - 1u)) << (4 * i);
        }
        R |= (uint32_t)__popc(S & ((1u << b) - 1u)) << (4 * (K - 1));
        ecode = 0;
        for (int e = 0; e < m; ++e) {
            const uint32_t ed = edge[e];
            const uint32_t ra = (R >> (4 * (ed & 15u))) & 15u;
            const uint32_t rb = (R >> (4 * (ed >> 4))) & 15u;
            const uint32_t lo = min(ra, rb), hi = max(ra, rb);
            const uint32_t p = lo * (2u * K - lo - 1u) / 2u + (hi - lo - 1u);
            ecode |= 1u << (eb - 1 - (int)p);
        }
    }
    return ((unsigned long long)s << (W + eb)) | ((unsigned long long)sb << eb) | ecode;
}

template <int W, int K>
__device__ __forceinline__ void consider(const Ctx &c, Best &bst, uint32_t S, unsigned long long fpack,
                                         uint32_t s) {
    const unsigned long long key = make_key<W, K>(S, fpack, (uint32_t)c.b, s, c.clique, c.eb, c.m, c.edge);
    if (key > bst.key) {
        bst.key = key;
        bst.bs = s;
    }
}

template <int K, int SEL, int J>
__device__ __forceinline__ St<K> push(const Ctx &c, const St<K> &st, uint32_t v) {
    St<K> s = st;
    const uint32_t vb = 1u << v;
    const uint4 t = c.cm[v];
    if constexpr (SEL == SEL_LIN) {
        const uint32_t X = c.useU ? st.U : st.bm[J];
        const int n12 = c.useU ? J : (int)((c.db >> (8 * J)) & 0xFFu);
        const int incv = c.useU ? c.inc[v] : 0;
        s.acc = st.acc + c.w12 * n12 - incv + c.w0 * __popc(t.x & X) + c.w1 * __popc(t.y & X) +
                c.w2 * __popc(t.z & X);
    } else {
        const uint32_t X = st.bm[J];
        s.acc = st.acc + __popc(t.x & X);
        s.acc2 = st.acc2 + __popc((t.y | t.z) & X);
    }
    s.U = st.U | vb;
    s.f[J] = v;
    const uint32_t fbJ = (uint32_t)(c.fb >> (8 * J)) & 0xFFu;
    const uint32_t fsJ = (uint32_t)(c.fs >> (8 * J)) & 0xFFu;
    const uint32_t above = 0xFFFFFFFEu << v;
#pragma unroll
    for (int u = J + 1; u < K; ++u) {
        if ((fbJ >> u) & 1u) s.bm[u] |= vb;
        if ((fsJ >> u) & 1u) s.al[u] &= above;
    }
    return s;
}

template <int K>
__device__ __forceinline__ unsigned long long pack_f(const St<K> &st) {
    unsigned long long fpack = 0;
#pragma unroll
    for (int i = 0; i < K - 1; ++i) fpack |= (unsigned long long)st.f[i] << (8 * i);
    return fpack;
}

// k = 1: a single level, the lanes are the devices of vertex 0.
template <int W, int SEL>
__device__ __forceinline__ void leaf_k1(const Ctx &c, Best &bst) {
    const bool act = (c.F >> c.b) & 1u;
    const int s = (SEL == SEL_LIN) ? c.acc0 + c.leafC : 0;  // m = 0: census (0,0,0) has rank 0
    bst.cnt += act ? 1u : 0u;
    if (act && (uint32_t)s >= bst.bs) consider<W, 1>(c, bst, 1u << c.b, 0ull, (uint32_t)s);
}

// The two innermost levels: vertex K-2 walks the devices of `cand`
// (uniform loop), vertex K-1 sits on the lanes.  Vertices 0..K-3 are placed.
template <int W, int K, int SEL>
__device__ __forceinline__ void inner(const Ctx &c, const St<K> &st, uint32_t cand, Best &bst) {
    constexpr int J = K - 2;
    const uint32_t b = (uint32_t)c.b;
    const uint32_t fbJ = (uint32_t)(c.fb >> (8 * J)) & 0xFFu;
    const uint32_t fsJ = (uint32_t)(c.fs >> (8 * J)) & 0xFFu;
    const bool eK = (fbJ >> (K - 1)) & 1u;   // pattern edge (K-2, K-1)
    const bool dep = (fsJ >> (K - 1)) & 1u;  // lex-leader f(K-2) < f(K-1)
    // (a) t2: increment of placing vertex K-2 on this lane's device;
    // (b) lp: this lane's leaf partial over vertices 0..K-3.
    int t2, base;
    if constexpr (SEL == SEL_LIN) {
        const uint32_t X2 = c.useU ? st.U : st.bm[J];
        const uint32_t X1 = c.useU ? st.U : st.bm[K - 1];
        const int n2 = c.useU ? J : (int)((c.db >> (8 * J)) & 0xFFu);
        t2 = c.w12 * n2 - (c.useU ? c.incb : 0) + c.w0 * __popc(c.cm0 & X2) + c.w1 * __popc(c.cm1 & X2) +
             c.w2 * __popc(c.cm2 & X2);
        const int lp = c.laneC + c.w12 * __popc(X1) + c.w0 * __popc(c.cm0 & X1) + c.w1 * __popc(c.cm1 & X1) +
                       c.w2 * __popc(c.cm2 & X1);
        base = (st.acc + lp + 1) * 32;
    } else {
        const uint32_t X2 = st.bm[J], X1 = st.bm[K - 1];
        t2 = __popc(c.cm0 & X2) * c.xs + __popc(c.cm12 & X2);
        base = (st.acc + __popc(c.cm0 & X1)) * c.xs + st.acc2 + __popc(c.cm12 & X1);  // census index
    }
    // Candidate list of this group, in increasing device order: entry i =
    // (byte offset of table row v, LIN rank increment 32*t2 + 31 - v,
    //  SENS census-index increment t2, 31 - v).
    const uint32_t n = (uint32_t)__popc(cand);
    __syncwarp(c.gmask);  // previous readers of the list are done
    if ((cand >> b) & 1u)
        c.list[__popc(cand & ((1u << b) - 1u))] = make_int4((int)b * 128, t2 * 32 + 31 - (int)b, t2, 31 - (int)b);
    __syncwarp(c.gmask);
    const bool laneok = ((c.F & ~st.U & st.al[K - 1]) >> b) & 1u;
    // leaves counted: v in cand with v != b (and v < b if canonical-ordered)
    const uint32_t M = laneok ? (dep ? ((1u << b) - 1u) : ~(1u << b)) : 0u;
    bst.cnt += (uint32_t)__popc(M & cand);
    // Within this call the lane's leaves differ only in v, and for equal
    // scores the smaller v is the lex-smaller device set (larger key): the
    // packed rank (score+1)*32 + 31-v is maxed branch-free and the full key
    // is built once afterwards.
    int best = 0;
    if constexpr (SEL == SEL_LIN) {
        const bool eW = c.w12 != 0 && (c.useU || eK);
        const char *tb = reinterpret_cast<const char *>((eW ? (dep ? c.twd : c.tw) : (dep ? c.tzd : c.tz)) + b);
#pragma unroll 4
        for (uint32_t i = 0; i < n; ++i) {
            const int4 e = c.list[i];
            best = max(best, base + e.y + *reinterpret_cast<const int *>(tb + e.x));
        }
    } else {
        const char *tz = reinterpret_cast<const char *>((dep ? c.tzd : c.tz) + b);
        if (eK) {
            const char *td = reinterpret_cast<const char *>(c.tdl + b);
#pragma unroll 4
            for (uint32_t i = 0; i < n; ++i) {
                const int4 e = c.list[i];
                const int idx = base + e.z + *reinterpret_cast<const int *>(td + e.x);
                best = max(best, (int)c.lut[idx] + e.w + *reinterpret_cast<const int *>(tz + e.x));
            }
        } else {
#pragma unroll 4
            for (uint32_t i = 0; i < n; ++i) {
                const int4 e = c.list[i];
                best = max(best, (int)c.lut[base + e.z] + e.w + *reinterpret_cast<const int *>(tz + e.x));
            }
        }
    }
    if (laneok && best >= 32) {
        const uint32_t s = (uint32_t)(best >> 5) - 1u;
        if (s >= bst.bs) {
            const uint32_t bestv = 31u - (uint32_t)(best & 31);
            unsigned long long fpack = pack_f<K>(st);
            fpack |= (unsigned long long)bestv << (8 * J);
            consider<W, K>(c, bst, st.U | (1u << bestv) | (1u << b), fpack, s);
        }
    }
}

template <int W, int K, int SEL, int J>
__device__ __forceinline__ void level(const Ctx &c, const St<K> &st, Best &bst) {
    if constexpr (K == 1) {
        leaf_k1<W, SEL>(c, bst);
    } else if constexpr (J == K - 2) {
        inner<W, K, SEL>(c, st, c.F & ~st.U & st.al[J], bst);
    } else {
        uint32_t cand = c.F & ~st.U & st.al[J];
        while (cand) {
            const uint32_t v = __ffs(cand) - 1;
            cand &= cand - 1u;
            level<W, K, SEL, J + 1>(c, push<K, SEL, J>(c, st, v), bst);
        }
    }
}

template <int K>
__device__ __forceinline__ St<K> root(const Ctx &c) {
    St<K> st;
    st.U = 0;
    st.acc = c.acc0;
    st.acc2 = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        st.f[i] = 0;
        st.bm[i] = 0;
        st.al[i] = kFull;
    }
    return st;
}

// item -> mixed-radix digits (radix nF - j at level j); false if item >= P(nF, D)
__device__ __forceinline__ bool digits(uint32_t item, int nF, int D, const uint32_t *magic,
                                       uint32_t (&dg)[kMaxDecode]) {
    uint32_t it = item;
#pragma unroll
    for (int j = kMaxDecode - 1; j >= 0; --j) {
        if (j < D) {
            const uint32_t r = (uint32_t)(nF - j);
            const uint32_t q = __umulhi(it, magic[r]);
            dg[j] = it - q * r;
            it = q;
        } else {
            dg[j] = 0;
        }
    }
    return it == 0;
}

__device__ __forceinline__ uint32_t perm_count(int n, int d) {
    uint32_t p = 1;
    for (int j = 0; j < d; ++j) p *= (uint32_t)(n - j);
    return p;
}

// Walk up to maxn consecutive items starting at the item whose digits are dg.
// Levels < D-1 are decoded from the digits; level D-1 iterates its (raw-order)
// candidates from digit dg[D-1] on.  Returns the number of items consumed
// (>= 1); a prefix that violates a lex-leader bound skips its whole subtree.
template <int W, int K, int SEL, int J, int DMAX>
__device__ __forceinline__ uint32_t descend_range(const Ctx &c, const St<K> &st, const uint32_t (&dg)[kMaxDecode],
                                                  int D, uint32_t maxn, Best &bst) {
    if constexpr (J >= DMAX || J > K - 2) {
        return maxn;  // unreachable: D <= DMAX <= K-1
    } else {
        if (J < D - 1) {
            const uint32_t v = nth_set(c.F & ~st.U, dg[J]);
            if (!((st.al[J] >> v) & 1u)) {
                uint32_t prod = 1, off = 0;
#pragma unroll
                for (int l = kMaxDecode - 1; l > J; --l) {
                    if (l < D) {
                        off += dg[l] * prod;
                        prod *= (uint32_t)(c.nF - l);
                    }
                }
                return min(maxn, prod - off);
            }
            return descend_range<W, K, SEL, J + 1, DMAX>(c, push<K, SEL, J>(c, st, v), dg, D, maxn, bst);
        } else {
            uint32_t cand = c.F & ~st.U;
            const uint32_t p = nth_set(cand, dg[J]);
            cand &= ~((1u << p) - 1u);  // raw candidates from the current item on
            uint32_t n = (uint32_t)__popc(cand);
            if (maxn < n) {
                cand &= (1u << nth_set(cand, maxn)) - 1u;
                n = maxn;
            }
            cand &= st.al[J];
            if constexpr (J == K - 2) {
                inner<W, K, SEL>(c, st, cand, bst);
            } else {
                while (cand) {
                    const uint32_t v = __ffs(cand) - 1;
                    cand &= cand - 1u;
                    level<W, K, SEL, J + 1>(c, push<K, SEL, J>(c, st, v), bst);
                }
            }
            return n;
        }
    }
}

// Items [lo, hi) of depth D (D = 0 only for K = 1).
template <int W, int K, int SEL, int DMAX>
__device__ __forceinline__ void run_range(const Ctx &c, uint32_t lo, uint32_t hi, int D, const uint32_t *magic,
                                          Best &bst) {
    if constexpr (K == 1) {
        if (lo == 0 && hi > 0) leaf_k1<W, SEL>(c, bst);
    } else {
        uint32_t i = lo;
        while (i < hi) {
            uint32_t dg[kMaxDecode];
            if (!digits(i, c.nF, D, magic, dg)) break;
            i += descend_range<W, K, SEL, 0, DMAX>(c, root<K>(c), dg, D, hi - i, bst);
        }
    }
}

// Per-query context.  Must be called by the whole warp (uses shuffles).
// s_inc: per-warp (or per-CTA) smem table of inc_F, written by group 0.
template <int W>
__device__ __forceinline__ Ctx make_ctx(const DevTopo &topo, const SmemTopo &sm, int *s_inc,
                                        const uint16_t *s_lut, int xs, int4 *s_list, const DevPattern &P,
                                        uint32_t busy, int selector, int sensitive) {
    const uint4 *s_cm = sm.cm;
    const int lane = threadIdx.x & 31;
    Ctx c;
    const uint32_t nmask = topo.n >= 32 ? kFull : ((1u << topo.n) - 1u);
    c.F = ~busy & nmask;
    c.nF = __popc(c.F);
    c.b = lane & (W - 1);
    const int g = lane / W;
    c.gmask = W == 32 ? kFull : (((1u << W) - 1u) << (g * W));
    const uint4 mine = s_cm[c.b];
    c.cm0 = mine.x;
    c.cm1 = mine.y;
    c.cm2 = mine.z;
    c.cm12 = mine.y | mine.z;
    // inc_F(b) = sum_{u in F, u != b} w(u,b)
    const int inFb = (c.F >> c.b) & 1u;
    int incb = 12 * (c.nF - inFb) + 38 * __popc(mine.x & c.F) + 13 * __popc(mine.y & c.F) +
               8 * __popc(mine.z & c.F);
    if (c.b >= topo.n) incb = 0;
    if (lane < W) s_inc[c.b] = incb;
    c.incb = incb;
    // T_F = 1/2 sum_{v in F} inc_F(v)  (reduce within the W-lane group)
    int t = inFb ? incb : 0;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o, W);
    const int TF = t / 2;
    const int K = P.k;
    c.fb = *reinterpret_cast<const uint64_t *>(P.fwd_back);
    c.fs = *reinterpret_cast<const uint64_t *>(P.fwd_src);
    c.db = *reinterpret_cast<const uint64_t *>(P.dback);
    c.clique = P.clique;
    c.eb = P.eb;
    c.m = P.m;
    c.edge = P.edge;
    c.mp1 = P.m + 1;
    c.cm = s_cm;
    c.inc = s_inc;
    c.lut = s_lut;
    c.xs = xs;
    c.tw = sm.tw;
    c.tz = sm.tz;
    c.twd = sm.twd;
    c.tzd = sm.tzd;
    c.tdl = sm.tdl;
    c.list = s_list + g * W;
    c.laneC = 0;
    if (selector == MAPA_SEL_BASELINE) {
        c.w0 = c.w1 = c.w2 = c.w12 = 0;
        c.useU = 0;
        c.acc0 = 0;
    } else if (selector == MAPA_SEL_PRESERVE && !sensitive) {  // Eq. 3
        c.w0 = 38; c.w1 = 13; c.w2 = 8; c.w12 = 12;
        c.useU = 1;
        c.acc0 = TF;
        c.laneC = -incb;
    } else {  // Eq. 1 (or Eq. 2 census for the sensitive kernel)
        c.w0 = 38; c.w1 = 13; c.w2 = 8; c.w12 = 12;
        c.useU = 0;
        c.acc0 = 0;
    }
    const int n12 = c.useU ? (K - 1) : (int)P.dback[K - 1];
    c.leafC = c.w12 * n12 + c.laneC;
    __syncwarp();
    return c;
}

__device__ __forceinline__ void warp_reduce(unsigned long long &key, unsigned long long &cnt) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(kFull, key, o);
        const unsigned long long c2 = __shfl_xor_sync(kFull, cnt, o);
        key = k2 > key ? k2 : key;
        cnt += c2;
    }
}

// Topology tables in shared memory (SmemTopo) for Eq. 2 table stride xs.
// Caller syncs.
__device__ __forceinline__ void load_topo(const DevTopo &topo, SmemTopo &sm, int xs) {
    const int tid = threadIdx.x;
    if (tid < kMaxN) sm.cm[tid] = make_uint4(topo.cm[tid][0], topo.cm[tid][1], topo.cm[tid][2], topo.cm[tid][3]);
    if (tid <= kMaxN) sm.magic[tid] = tid >= 2 ? (0xFFFFFFFFu / (uint32_t)tid + 1u) : 0u;
    for (int i = tid; i < kMaxN * kMaxN; i += blockDim.x) {
        const int v = i >> 5, b = i & 31;
        int w = kNeg, d = 0;
        if (v != b && v < topo.n && b < topo.n) {
            if ((topo.cm[b][0] >> v) & 1u) { w = 50; d = xs; }
            else if ((topo.cm[b][1] >> v) & 1u) { w = 25; d = 1; }
            else if ((topo.cm[b][2] >> v) & 1u) { w = 20; d = 1; }
            else w = 12;
        }
        const int z = w == kNeg ? kNeg : 0;
        const int wv = w == kNeg ? kNeg : 32 * w;
        sm.tw[i] = wv;
        sm.tz[i] = z;
        sm.twd[i] = v >= b ? kNeg : wv;
        sm.tzd[i] = v >= b ? kNeg : z;
        sm.tdl[i] = d;
    }
}

// Eq. 2 table for the kernels: out[x*xs + y] = (rank(x,y) + 1) * 32 from the
// host's dense rank table rank[x*(m+1) + y] (x + y <= m); other entries 0.
__device__ __forceinline__ void load_lut(const uint16_t *rank, int m, int xs, uint16_t *out) {
    for (int i = threadIdx.x; i < xs * xs; i += blockDim.x) {
        const int x = i / xs, y = i % xs;
        out[i] = (x + y <= m) ? (uint16_t)((rank[x * (m + 1) + y] + 1) * 32) : (uint16_t)0;
    }
}

// ---------------------------------------------------------------- single query
// Items = prefixes of depth D, in chunks of `chunk` consecutive items; local
// chunk q of rank r is global chunk q*world + r.  Group g of a warp walks the
// g-th slice of the chunk.
template <int W, int K, int SEL>
__global__ void __launch_bounds__(kBlock, 2)
esa_single(const __grid_constant__ SingleTables tb, int selector, int sensitive,
           const mapa_query *__restrict__ dq, mapa_record *__restrict__ rec, int D, int rank,
           int world, int chunk) {
    constexpr int G = 32 / W;
    constexpr int DMAX = (K - 1) < kMaxDecode ? (K - 1) : kMaxDecode;
    __shared__ SmemTopo s_topo;
    __shared__ int s_inc[kMaxN];
    __shared__ uint16_t s_lut[kLutCapSingle];
    __shared__ uint8_t s_edge[28];
    __shared__ int4 s_list[kWarps][32];
    __shared__ unsigned long long s_key[kWarps], s_cnt[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DevPattern &P = tb.pat[0];
    const int xs = P.m <= 15 ? 16 : 32;
    load_topo(tb.topo, s_topo, xs);
    load_lut(tb.lut + P.lut_off, P.m, xs, s_lut);
    if (tid < 28) s_edge[tid] = P.edge[tid];
    const uint32_t *s_magic = s_topo.magic;
    const uint32_t busy = dq->busy;
    __syncthreads();

    Ctx c = make_ctx<W>(tb.topo, s_topo, s_inc, s_lut, xs, s_list[warp], P, busy, selector, sensitive);
    c.edge = s_edge;
    __syncthreads();  // s_inc written by every warp with identical values

    const uint32_t nItems = (K <= c.nF) ? perm_count(c.nF, D) : 0u;
    const uint32_t nChunks = (nItems + (uint32_t)chunk - 1u) / (uint32_t)chunk;
    const uint32_t per = (uint32_t)chunk / G;  // host makes chunk a multiple of G
    Best bst{0ull, 0u, 0u};
    const uint32_t g = (uint32_t)(lane / W);
    for (;;) {
        uint32_t q = 0;
        if (lane == 0) q = atomicAdd(&rec->ctr, 1u);
        q = __shfl_sync(kFull, q, 0);
        const uint32_t gq = q * (uint32_t)world + (uint32_t)rank;
        if (gq >= nChunks) break;
        const uint32_t lo = gq * (uint32_t)chunk + g * per;
        const uint32_t hi = min(lo + per, nItems);
        if (lo < hi) run_range<W, K, SEL, DMAX>(c, lo, hi, D, s_magic, bst);
        __syncwarp();
    }
    unsigned long long key = bst.key, cnt = bst.cnt;
    warp_reduce(key, cnt);
    if (lane == 0) {
        s_key[warp] = key;
        s_cnt[warp] = cnt;
    }
    __syncthreads();
    if (warp == 0) {
        key = lane < kWarps ? s_key[lane] : 0ull;
        cnt = lane < kWarps ? s_cnt[lane] : 0ull;
        warp_reduce(key, cnt);
        if (lane == 0) {
            if (key) atomicMax(u64p(&rec->key), key);
            if (cnt) atomicAdd(u64p(&rec->leaves), cnt);
        }
    }
}

// ---------------------------------------------------------------- batches
// W slots per query; slot j = the j-th free device as f(0) (items of depth 1);
// K = 1 queries use slot 0 only (depth 0).
template <int W, int K, int SEL>
__device__ __forceinline__ void batch_item(const Ctx &c, uint32_t j, const uint32_t *magic, Best &bst) {
    if constexpr (K == 1) {
        if (j == 0) leaf_k1<W, SEL>(c, bst);
    } else {
        if (j < (uint32_t)c.nF) run_range<W, K, SEL, 1>(c, j, j + 1, 1, magic, bst);
    }
}

template <int W, int SEL>
__device__ __forceinline__ void batch_dispatch_k(int K, const Ctx &c, uint32_t j, const uint32_t *magic,
                                                 Best &bst) {
    switch (K) {
        case 1: batch_item<W, 1, SEL>(c, j, magic, bst); break;
        case 2: batch_item<W, 2, SEL>(c, j, magic, bst); break;
        case 3: batch_item<W, 3, SEL>(c, j, magic, bst); break;
        case 4: batch_item<W, 4, SEL>(c, j, magic, bst); break;
        case 5: batch_item<W, 5, SEL>(c, j, magic, bst); break;
        case 6: batch_item<W, 6, SEL>(c, j, magic, bst); break;
        case 7: batch_item<W, 7, SEL>(c, j, magic, bst); break;
        case 8: batch_item<W, 8, SEL>(c, j, magic, bst); break;
        default: break;
    }
}

__device__ __forceinline__ bool key_fits(int W, const DevPattern &P) { return 15 + W + P.eb <= 63; }

template <int W>
__global__ void __launch_bounds__(kBlock, 2)
esa_batch(const __grid_constant__ MultiTables tb, long long nq, const mapa_query *__restrict__ qs,
          mapa_record *__restrict__ res, uint32_t *__restrict__ ctr) {
    constexpr int G = 32 / W;
    __shared__ SmemTopo s_topo;
    __shared__ int s_inc[kWarps][kMaxN];
    __shared__ int4 s_list[kWarps][32];
    extern __shared__ uint16_t s_lut[];  // npats * xs * xs Eq. 2 tables (dynamic)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int xs = tb.xs;
    load_topo(tb.topo, s_topo, xs);
    for (int p = 0; p < tb.npats; ++p) load_lut(tb.lut + tb.pat[p].lut_off, tb.pat[p].m, xs, s_lut + p * xs * xs);
    const uint32_t *s_magic = s_topo.magic;
    __syncthreads();

    const unsigned long long nslots = (unsigned long long)nq * W;
    const uint32_t g = (uint32_t)(lane / W);
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(reinterpret_cast<unsigned long long *>(ctr), (unsigned long long)G);
        base = __shfl_sync(kFull, base, 0);
        if (base >= nslots) break;
        const unsigned long long q = base / W;  // G | W: every group of the warp has the same query
        const mapa_query qu = qs[q];
        const uint32_t pid = qu.pattern;
        if (pid >= (uint32_t)tb.npats || !key_fits(W, tb.pat[pid < (uint32_t)tb.npats ? pid : 0])) {
            if (lane == 0 && (base % W) == 0) atomicExch(&res[q].status, 1u);
            continue;
        }
        const DevPattern &P = tb.pat[pid];
        Ctx c = make_ctx<W>(tb.topo, s_topo, s_inc[warp], s_lut + pid * xs * xs, xs, s_list[warp], P, qu.busy,
                            qu.selector, qu.sensitive);
        if (P.k > c.nF) continue;
        const uint32_t j = (uint32_t)(base % W) + g;
        Best bst{0ull, 0u, 0u};
        const bool sens = qu.selector == MAPA_SEL_PRESERVE && qu.sensitive;
        if (sens) batch_dispatch_k<W, SEL_SENS>(P.k, c, j, s_magic, bst);
        else batch_dispatch_k<W, SEL_LIN>(P.k, c, j, s_magic, bst);
        __syncwarp();
        unsigned long long key = bst.key, cnt = bst.cnt;
        warp_reduce(key, cnt);
        if (lane == 0) {
            if (key) atomicMax(u64p(&res[q].key), key);
            if (cnt) atomicAdd(u64p(&res[q].leaves), cnt);
        }
    }
}

// ---------------------------------------------------------------- trace replay
template <int W, int K, int SEL>
__device__ __forceinline__ void trace_items(const Ctx &c, int D, uint32_t nItems, uint32_t gid, uint32_t ngroups,
                                            const uint32_t *magic, Best &bst) {
    constexpr int DMAX = (K - 1) < 2 ? (K - 1) : 2;
    const uint32_t per = (nItems + ngroups - 1u) / ngroups;
    const uint32_t lo = gid * per, hi = min(lo + per, nItems);
    if (lo < hi) run_range<W, K, SEL, DMAX>(c, lo, hi, D, magic, bst);
}

template <int W, int SEL>
__device__ __forceinline__ void trace_dispatch_k(int K, const Ctx &c, int D, uint32_t nItems, uint32_t gid,
                                                 uint32_t ngroups, const uint32_t *magic, Best &bst) {
    switch (K) {
        case 1: trace_items<W, 1, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        case 2: trace_items<W, 2, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        case 3: trace_items<W, 3, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        case 4: trace_items<W, 4, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        case 5: trace_items<W, 5, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        case 6: trace_items<W, 6, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        case 7: trace_items<W, 7, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        case 8: trace_items<W, 8, SEL>(c, D, nItems, gid, ngroups, magic, bst); break;
        default: break;
    }
}

// One CTA per trace; ALLOC / RELEASE ops in order; the busy mask lives in
// shared memory (§3.6 state management), decisions go to HBM as keys.
template <int W>
__global__ void __launch_bounds__(kBlock, 1)
esa_trace(const __grid_constant__ MultiTables tb, int nops, const mapa_trace_op *__restrict__ ops, int njobs,
          const mapa_query *__restrict__ jobs, unsigned long long *__restrict__ keys) {
    constexpr int G = 32 / W;
    __shared__ SmemTopo s_topo;
    __shared__ int s_inc[kWarps][kMaxN];
    __shared__ int4 s_list[kWarps][32];
    __shared__ unsigned long long s_key[kWarps];
    __shared__ uint32_t s_busy;
    extern __shared__ uint16_t s_lut[];  // npats * xs * xs Eq. 2 tables (dynamic)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x;
    const int xs = tb.xs;
    load_topo(tb.topo, s_topo, xs);
    for (int p = 0; p < tb.npats; ++p) load_lut(tb.lut + tb.pat[p].lut_off, tb.pat[p].m, xs, s_lut + p * xs * xs);
    const uint32_t *s_magic = s_topo.magic;
    if (tid == 0) s_busy = 0u;
    __syncthreads();
    const mapa_trace_op *op = ops + (long long)t * nops;
    const mapa_query *jb = jobs + (long long)t * njobs;
    unsigned long long *ky = keys + (long long)t * njobs;
    const uint32_t gid = (uint32_t)(warp * G + lane / W);
    const uint32_t wmask = W >= 32 ? kFull : ((1u << W) - 1u);
    for (int o = 0; o < nops; ++o) {
        const mapa_trace_op cur = op[o];
        const mapa_query qu = jb[cur.job];
        const uint32_t pid = qu.pattern;
        const bool okp = pid < (uint32_t)tb.npats && key_fits(W, tb.pat[pid < (uint32_t)tb.npats ? pid : 0]);
        const DevPattern &P = tb.pat[okp ? pid : 0];
        if (cur.op == 0) {
            const uint32_t busy = s_busy;
            Ctx c = make_ctx<W>(tb.topo, s_topo, s_inc[warp], s_lut + (okp ? pid : 0) * xs * xs, xs, s_list[warp], P,
                                busy, qu.selector, qu.sensitive);
            Best bst{0ull, 0u, 0u};
            if (okp && P.k <= c.nF) {
                const int D = (P.k - 1) < 2 ? (P.k - 1) : 2;
                const uint32_t nItems = perm_count(c.nF, D);
                const bool sens = qu.selector == MAPA_SEL_PRESERVE && qu.sensitive;
                if (sens) trace_dispatch_k<W, SEL_SENS>(P.k, c, D, nItems, gid, kWarps * G, s_magic, bst);
                else trace_dispatch_k<W, SEL_LIN>(P.k, c, D, nItems, gid, kWarps * G, s_magic, bst);
            }
            __syncwarp();
            unsigned long long key = bst.key, cnt = bst.cnt;
            warp_reduce(key, cnt);
            if (lane == 0) s_key[warp] = key;
            __syncthreads();
            if (tid == 0) {
                unsigned long long best = 0;
                for (int w = 0; w < kWarps; ++w) best = s_key[w] > best ? s_key[w] : best;
                ky[cur.job] = best;
                if (best) s_busy = busy | (__brev((uint32_t)(best >> P.eb) & wmask) >> (32 - W));
            }
        } else {
            if (tid == 0) {
                const unsigned long long kk = ky[cur.job];
                s_busy &= ~(__brev((uint32_t)(kk >> P.eb) & wmask) >> (32 - W));
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- dispatch tables
template <int W, int K, int SEL>
int do_launch_single(const SingleTables &tb, int selector, int sensitive, const mapa_query *dq,
                     mapa_record *rec, int D, int rank, int world, int chunk, int grid, cudaStream_t st) {
    esa_single<W, K, SEL><<<grid, kBlock, 0, st>>>(tb, selector, sensitive, dq, rec, D, rank, world, chunk);
    return (int)cudaGetLastError();
}

using SingleFn = int (*)(const SingleTables &, int, int, const mapa_query *, mapa_record *, int, int, int,
                         int, int, cudaStream_t);

template <int W, int SEL>
SingleFn pick_k(int K) {
    switch (K) {
        case 1: return do_launch_single<W, 1, SEL>;
        case 2: return do_launch_single<W, 2, SEL>;
        case 3: return do_launch_single<W, 3, SEL>;
        case 4: return do_launch_single<W, 4, SEL>;
        case 5: return do_launch_single<W, 5, SEL>;
        case 6: return do_launch_single<W, 6, SEL>;
        case 7: return do_launch_single<W, 7, SEL>;
        case 8: return do_launch_single<W, 8, SEL>;
    }
    return nullptr;
}

template <int W>
SingleFn pick_sel(int K, int sens) {
    return sens ? pick_k<W, SEL_SENS>(K) : pick_k<W, SEL_LIN>(K);
}

SingleFn pick_single(int W, int K, int sens) {
    if (W == 8) return pick_sel<8>(K, sens);
    if (W == 16) return pick_sel<16>(K, sens);
    if (W == 32) return pick_sel<32>(K, sens);
    return nullptr;
}

template <int W, int K, int SEL>
const void *single_ptr() { return (const void *)esa_single<W, K, SEL>; }

}  // namespace

int launch_single(const SingleTables &tb, int selector, int sensitive, const mapa_query *d_query,
                  mapa_record *d_record, int depth, int rank, int world, int chunk, int grid, void *stream) {
    const int sensk = (selector == MAPA_SEL_PRESERVE && sensitive) ? 1 : 0;
    SingleFn fn = pick_single(tb.topo.width, tb.pat[0].k, sensk);
    if (!fn) return (int)cudaErrorInvalidValue;
    return fn(tb, selector, sensitive, d_query, d_record, depth, rank, world, chunk, grid,
              (cudaStream_t)stream);
}

int launch_batch(const MultiTables &tb, int64_t nq, const mapa_query *d_queries, mapa_record *d_results,
                 uint32_t *d_ctr, int grid, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int dyn = tb.npats * tb.xs * tb.xs * (int)sizeof(uint16_t);
    switch (tb.topo.width) {
        case 8: esa_batch<8><<<grid, kBlock, dyn, st>>>(tb, (long long)nq, d_queries, d_results, d_ctr); break;
        case 16: esa_batch<16><<<grid, kBlock, dyn, st>>>(tb, (long long)nq, d_queries, d_results, d_ctr); break;
        case 32: esa_batch<32><<<grid, kBlock, dyn, st>>>(tb, (long long)nq, d_queries, d_results, d_ctr); break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)cudaGetLastError();
}

int launch_trace(const MultiTables &tb, int ntraces, int nops, const mapa_trace_op *d_ops, int njobs,
                 const mapa_query *d_jobs, uint64_t *d_keys, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *k = reinterpret_cast<unsigned long long *>(d_keys);
    const int dyn = tb.npats * tb.xs * tb.xs * (int)sizeof(uint16_t);
    switch (tb.topo.width) {
        case 8: esa_trace<8><<<ntraces, kBlock, dyn, st>>>(tb, nops, d_ops, njobs, d_jobs, k); break;
        case 16: esa_trace<16><<<ntraces, kBlock, dyn, st>>>(tb, nops, d_ops, njobs, d_jobs, k); break;
        case 32: esa_trace<32><<<ntraces, kBlock, dyn, st>>>(tb, nops, d_ops, njobs, d_jobs, k); break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)cudaGetLastError();
}

int device_sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

namespace {
template <int W>
int occ_single(int K, int sens) {
    const void *f = nullptr;
#define MAPA_OCC_CASE(KK)                                                        \
    case KK:                                                                     \
        f = sens ? single_ptr<W, KK, SEL_SENS>() : single_ptr<W, KK, SEL_LIN>(); \
        break;
    switch (K) {
        MAPA_OCC_CASE(1) MAPA_OCC_CASE(2) MAPA_OCC_CASE(3) MAPA_OCC_CASE(4)
        MAPA_OCC_CASE(5) MAPA_OCC_CASE(6) MAPA_OCC_CASE(7) MAPA_OCC_CASE(8)
    }
#undef MAPA_OCC_CASE
    int nb = 0;
    if (!f || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kBlock, 0) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}
}  // namespace

int max_blocks_per_sm_single(int width, int k, int sens) {
    if (width == 8) return occ_single<8>(k, sens);
    if (width == 16) return occ_single<16>(k, sens);
    return occ_single<32>(k, sens);
}

int max_blocks_per_sm_batch(int width, int dyn_smem) {
    int nb = 0;
    cudaError_t e = cudaErrorInvalidValue;
    if (width == 8) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, esa_batch<8>, kBlock, dyn_smem);
    if (width == 16) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, esa_batch<16>, kBlock, dyn_smem);
    if (width == 32) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, esa_batch<32>, kBlock, dyn_smem);
    return (e == cudaSuccess && nb > 0) ? nb : 1;
}

int set_dynamic_smem(int bytes) {
    // batch / trace kernels keep npats Eq. 2 tables in dynamic shared memory
    const void *fs[6] = {(const void *)esa_batch<8>, (const void *)esa_batch<16>, (const void *)esa_batch<32>,
                         (const void *)esa_trace<8>, (const void *)esa_trace<16>, (const void *)esa_trace<32>};
    for (const void *f : fs) {
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return (int)e;
    }
    return 0;
}

const char *cuda_error_string(int err) { return cudaGetErrorString((cudaError_t)err); }

}  // namespace mapa
