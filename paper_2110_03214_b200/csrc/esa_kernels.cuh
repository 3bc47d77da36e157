// esa_kernels.cuh — Enumerate-Score-Argmax kernels for sm_100a (B200).
// Template code; instantiated per topology width W by esa_w8.cu / esa_w16.cu /
// esa_w32.cu (compiled in parallel) and dispatched by esa.cu.
//
// One pass = SURVEY.md §8(a) S3-S6 fused in registers / shared memory:
//   S3 occupancy prep   F = ~busy; inc_F(v), T_F (Eq. 3 support)
//   S4 enumeration      DFS over injective maps f: V(P) -> F (§3.3 P:496-501;
//                       G complete, so every injective map embeds).
//                       Lanes = devices of the LAST pattern vertex k-1; the
//                       two levels above it (k-3, k-2) walk per-group smem
//                       candidate lists; outer levels are a uniform DFS.
//                       Groups of W lanes (W = 8/16/32 = padded N) each run
//                       their own prefix, so small topologies fill the warp.
//                       Canonical mode adds lex-leader lower bounds (one leaf
//                       per Aut(P)-orbit = SPEC dedup S:209).
//   S5 scoring          integer only.  With v's class masks c0..c2 and any
//                       device set X not containing v:
//                         sum_{u in X} w(u,v) = 12|X| + 38 popc(c0&X)
//                                               + 13 popc(c1&X) + 8 popc(c2&X)
//                       (popc on the outer levels only).  For the inner levels
//                       the lanes precompute in parallel the increment of
//                       placing vertex k-3 / k-2 on their device (broadcast
//                       through the lists) and their own leaf partial; a
//                       k-3 step then costs one weight lookup per lane, a
//                       k-2 step one list read + one table read + one fused
//                       add-max per leaf.
//                         Eq. 1 AggBW: X = back-neighbour devices.
//                         Eq. 3 PreservedBW: T_F - sum inc_F(S)
//                         + inside(S), X = all placed devices.
//                         Eq. 2: census (x, y) accumulated as a
//                         table index x*xs + y; score = dense rank of Eq. 2
//                         among the censuses with x+y+z = m (host table).
//   S6 argmax           leaves of one k-2 scan are ranked by (score+1)*32 +
//                       (31 - v) (ties -> smaller v = lex-smaller device set);
//                       the packed 64-bit key (score | brev(S) | edge code) is
//                       built out of line only when a scan's best reaches the
//                       lane's best score; warp shuffle max, block max,
//                       atomicMax in HBM.  Max is order independent, so the
//                       result is identical for every grid size / rank count.
// Work items: the prefixes of depth D (mixed radix over the free devices),
// handed out as contiguous chunks; a chunk is walked as a DFS range, so only
// the first item of a run is decoded.  All tables live in one dynamic
// shared-memory block (Shared below) addressed by offset, so the per-query
// context holds no pointers.  No dense contraction exists, so no tensor cores
// are used; the bound is integer issue / LSU.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "internal.h"

namespace mapa {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kMaxDecode = 4;
constexpr int kNN = kMaxN * kMaxN;

// Compile-time selector: Greedy (Eq. 1), Preserve-insensitive (Eq. 3),
// Preserve-sensitive (Eq. 2 rank), Baseline (constant score).
// Bit 2 of the code = canonical mode (lex-leader constraints live); RAW-mode
// instantiations compile every constraint test away.
template <int SEL>
struct SelT {
    static constexpr int base = SEL & 3;
    static constexpr bool canon = (SEL & 4) != 0;
    static constexpr bool multi = (SEL & 8) != 0;      // batch / trace kernels (many patterns per block)
    // bit 4: branch-and-bound mode (MAPA_F_PRUNE, single-query kernels, k >= 4):
    // a k-2 scan runs only if an upper bound of its leaves reaches the best
    // score found so far by any lane of the grid (exact: the argmax is unchanged)
    static constexpr bool prune = (SEL & 16) != 0;
    // single-query Eq. 2 scans use 16-bit packed tables and columns (pack16)
    static constexpr bool pack16 = base == SEL_SENS && !multi;
    static constexpr bool lin = base != SEL_SENS;      // additive score (Eq. 1 / Eq. 3 / 0)
    // bit 5: single-query Eq. 1 / Eq. 3 scans on 16-bit lanes (two leaves per
    // VIADDMNMX.S16x2); the host sets it only when every scan value fits s16
    // (lin16_fits in mapa_host.cpp)
    // (batch kernels too: esa_batch picks it per query, from the query's own
    // free set; the trace kernel never sets bit 5)
    static constexpr bool lin16 = (SEL & 32) != 0 && lin;
    static constexpr bool half = pack16 || lin16;      // 16-bit table entries
    // single-query additive kernels share the CTA's best score as the hit
    // threshold (Shared::cthr, folded into the lane's Best::thr at each inner3
    // call; measured: Eq. 1 / 3 -6 % instructions; the Eq. 2 kernel, at the
    // 128-register cap, compiled to +15 % instructions with it, so it keeps
    // the lane's own threshold)
    static constexpr bool cta = lin && !multi;
    // single-query 16-bit kernels outside prune mode walk the two innermost
    // levels on static tables (inner3s / inners): per v3 the scan reads the
    // k-3 -> k-2 edge row of a table built once per CTA, and the lane's
    // column is re-based once per k-3 prefix, so no per-v3 table is built
    static constexpr bool stat = (pack16 || lin16) && !prune && !multi;
    static constexpr bool useU = base == SEL_INSENS;   // Eq. 3 sums over every placed device
    static constexpr int wt = base == SEL_BASE ? 0 : 1;
    static constexpr int w0 = 38 * wt, w1 = 13 * wt, w2 = 8 * wt, w12 = 12 * wt;
};

// Leaves of a k-2 scan are ranked by one int: (score + 1) * 32 + (31 - v).
// Invalid leaves (vertex k-1 on the device of k-2, a lex-leader violation,
// a padding lane) get kNeg added through the tables.
constexpr int kNeg = kNegTable;

// Per-warp candidate lists of the innermost DFS levels (G groups x W).
struct WarpLists {
    int dense[2][32];  // level k-2 (two v3 at a time): per device, increment of placing k-2 there (or a sentinel)
    int2 l3[32];    // level k-3: (v, increment of placing k-3 on v)
};

// One dynamic shared-memory block per CTA.  Tables are indexed [v*32 + b]:
//   tw  = 32 w(v,b), kNeg when v == b or either is not a device
//   tz  = 0,         kNeg likewise
//   twd / tzd = the same with kNeg also where v >= b (canonical f(k-2) < f(k-1))
//   twp = w(v,b) (0 when invalid), tdl = census delta xs [double] + [single]
//   tse / tsed = tdl + kSent when invalid (/ v >= b); ts0 / ts0d = 0 + kSent
//     (kSent = xs*xs moves the Eq. 2 index into a region of kNeg entries)
// followed by npats Eq. 2 tables of 3 xs^2 ints: [x*xs + y] = (rank+1)*32,
// [xs^2, 3 xs^2) = kNeg (an index carries at most two kSent offsets).
struct Shared {
    uint4 cm[kMaxN];
    uint32_t magic[kMaxN + 4];
    int tw[kNN], tz[kNN], twd[kNN], tzd[kNN], twp[kNN], tdl[kNN];
    int tse[kNN], tsed[kNN], ts0[kNN], ts0d[kNN];
    int inc[kWarps][kMaxN];
    WarpLists wl[kWarps];
    unsigned long long key[kWarps], cnt[kWarps];
    uint8_t edge[kMaxPats][28];
    uint32_t busy;
    int one;  // = 1 (Ctx::one)
    uint32_t topoS;  // trace kernel: the Topo-aware device set of the current ALLOC
    int cthr;        // single-query kernels: the CTA's best packed threshold (score + 1) * 32 so far
    unsigned long long ckey;  // single-query Eq. 2 kernels: the CTA's best key so far (sens_hit)
};

// Single-query kernels: Shared + one Eq. 2 table of 3 xs^2 ints + the
// prune-mode bound table of xs^2 ints, xs <= 40.
constexpr int kSmemSingleMax = (int)sizeof(Shared) + 4 * 40 * 40 * (int)sizeof(int);

extern __shared__ __align__(16) unsigned char g_smem[];
__device__ __forceinline__ Shared &sh() { return *reinterpret_cast<Shared *>(g_smem); }
__device__ __forceinline__ int *sh_lut() { return reinterpret_cast<int *>(g_smem + sizeof(Shared)); }

// Single-query Eq. 2 kernels (SelT::pack16) keep their one Eq. 2 table (and
// the prune-mode bound table) in STATIC shared memory: the first static
// variable of a kernel sits at the bottom of the CTA's shared window, shared
// address kLut1Addr, so the hot gathers address it as LDS [R + kLut1Addr]
// with the byte offset alone in R -- no per-leaf add of the window base, which
// the compiler otherwise keeps in a vector register under the 128-register
// cap (33 extra IMADs per scan, measured).  esa_single checks the address at
// run time and refuses the query (status 2) if it ever differs.
constexpr int kLut1Ints = 4 * 40 * 40;
constexpr uint32_t kLut1Addr = 0x400;
// Static tables of the SelT::stat kernels (W <= 32, pairs packed per word):
//   row[v3 * W/2 + q]: the entries of placing vertex k-2 on v = 2q / 2q+1 that
//     depend on v3 alone -- the (k-3, k-2) edge term and the sentinels of
//     v == v3 and of the lex-leader bound f(k-3) < f(k-2); row W is all zero
//     (the k-2-level scan of inners)
//   col[q * W + b]: lane b's column (edge (k-2, k-1) term, 31 - v tie-break for
//     additive scores, sentinels of v == b and of f(k-2) < f(k-1))
// The Eq. 2 kernels keep the LUT in front (StatSharedL, g_stL), the additive
// ones only the row / column tables (g_stN, no LUT: 4 KB, so three CTAs fit an
// SM); a kernel references one of the two, which sits at kLut1Addr.
struct StatTabs {
    uint32_t row[(32 + 1) * 16];
    uint32_t col[16 * 32];
};
struct StatSharedL {
    int lut[kLut1Ints];  // first: at kLut1Addr
    StatTabs t;
};
__shared__ __align__(16) StatSharedL g_stL;
__shared__ __align__(16) StatTabs g_stN;
// the Eq. 2 kernels' LUT (at kLut1Addr)
__device__ __forceinline__ int *lut1() { return g_stL.lut; }
template <bool L>
__device__ __forceinline__ StatTabs &stt() {
    if constexpr (L) return g_stL.t;
    else return g_stN;
}
template <bool L>
__device__ __forceinline__ const void *stat_base() {
    if constexpr (L) return &g_stL;
    else return &g_stN;
}
// 16-byte load of the static row table at byte offset `off` (immediate window
// address, as lds_lut1: a run-time window base would be rebuilt every iteration)
template <bool L>
__device__ __forceinline__ uint4 lds_row(uint32_t off) {
    constexpr int addr = (int)kLut1Addr + (L ? (int)offsetof(StatSharedL, t) : 0) + (int)offsetof(StatTabs, row);
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(off), "n"(addr));
    return v;
}
// lin16 sentinels of the static path: T2B (per prefix) / row / column.  Valid
// T2B entries are 32 (t2 + ishift) <= kStTmax, valid row entries 32 w <= 1600,
// valid column entries 32 w + 31 - v <= 1631: a valid leaf sums to
// [0, kStTmax + 3231]; any sentinel makes the sum negative (each dominates the
// other two's valid maximum) and the three together stay >= -32768.
constexpr int kStX = -3232, kStY = -14768, kStZ = -14768;
constexpr int kStTmax = kLin16StatMax;
static_assert(kStTmax == -kStY - 1632 && kStTmax == -kStZ - 1632, "see kLin16StatMax");
static_assert(-(kStX + kStY + kStZ) <= 32768, "s16 range");

// gather at byte offset `off` of lut1() (volatile: never merged with another
// load, so no gathered value is kept live across the hit branch)
__device__ __forceinline__ int lds_lut1(uint32_t off) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1+1024];" : "=r"(v) : "r"(off));
    return v;
}
static_assert(kLut1Addr == 1024, "lds_lut1 immediate");

template <int W>
struct Ctx {
    uint32_t F;
    int nF;
    int b;                          // lane's device id (lane % W)
    int g;                          // lane's group in the warp
    int warp;
    uint32_t gmask;                 // lanes of this lane's group
    uint32_t cm0, cm1, cm2, cm12;   // lane's class masks
    int incb;                       // inc_F(b)
    int laneC;                      // lane constant of the score (Eq. 3: -inc_F(b))
    int leafC;                      // k = 1 leaf constant
    int acc0;                       // accumulator at the root (T_F for Eq. 3)
    int xs;                         // Eq. 2 table row stride (16 or 32)
    int lut;                        // this pattern's Eq. 2 table offset (ints) in sh_lut()
    int pid;                        // pattern index (edge list in smem)
    uint64_t fb, fs, db;            // bytes: fwd_back, fwd_src, dback
    int clique, eb, m;
    int one;                        // 1, read from shared memory (see scan_dense)
    int negk;                       // -65536 at run time (pack16 offset split on the FMA pipe)
    int colmax;                     // additive scores: max_v col[v] (prune-mode bound)
    int ishift;                     // lin16 Eq. 3: max_{v in F} inc_F(v), added to table entries (0 otherwise)
    int irange;                     // lin16 Eq. 3: ishift - min_{v in F} inc_F(v)
    int col[W];                     // lane's inner-scan column (see lane_column)
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
    uint32_t bs;   // score of key
    uint32_t cnt;  // leaves scored
    int thr;       // (bs + 1) * 32: a scan's packed rank must reach this to matter
    uint32_t sb;   // brev_W(device set) of key (0 while no key)
    int pthr;      // prune mode: max(thr, 32 * (grid-wide best score + 1))
    unsigned *gb;  // prune mode: grid-wide best score + 1 (in the result record), else null
};

template <int SEL>
__device__ __forceinline__ uint32_t alw(uint32_t al) { return SelT<SEL>::canon ? al : 0xFFFFFFFFu; }

__device__ __forceinline__ unsigned long long *u64p(uint64_t *p) {
    return reinterpret_cast<unsigned long long *>(p);
}

__device__ __forceinline__ int lds_off(const int *base, int byte_off) {
    return *reinterpret_cast<const int *>(reinterpret_cast<const char *>(base) + byte_off);
}

// a * b + c that the compiler may not re-associate (the pack16 low-half
// offset: re-associated, the shared-window base costs one add per leaf
// instead of riding in the uniform operand of LDS [R+UR+imm])
__device__ __forceinline__ int mad_lo(int a, int b, int c) {
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
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

// Packed argmax key: score | brev_W(S) | edge code, built
// out of line on the slow path; arguments by value.
//   fpack: f(0..K-2) one byte each; b: device of vertex K-1.
template <int W, int K>
__device__ __noinline__ unsigned long long make_key(uint32_t S, unsigned long long fpack, uint32_t b,
                                                    uint32_t s, int clique, int eb, int m, int pid) {
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
        const uint8_t *edge = sh().edge[pid];
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

// Called when a leaf's score s >= the lane's best score.  An equal score wins
// only through the device-set field (brev_W(S), kept in a register), or, for
// the same set of a non-clique pattern, through the edge code.
template <int W, int K, bool CTA = false, bool CKEY = false>
__device__ __forceinline__ void consider(const Ctx<W> &c, Best &bst, uint32_t S, unsigned long long fpack,
                                         uint32_t s) {
    const uint32_t sbn = __brev(S) >> (32 - W);
    if (s == bst.bs && (sbn < bst.sb || (sbn == bst.sb && c.clique))) return;
    const unsigned long long key = make_key<W, K>(S, fpack, (uint32_t)c.b, s, c.clique, c.eb, c.m, c.pid);
    if (key > bst.key) {
        bst.key = key;
        bst.bs = s;
        bst.thr = ((int)s + 1) * 32;
        bst.sb = sbn;
        if constexpr (CTA) atomicMax(&sh().cthr, bst.thr);  // the CTA's threshold (see inner3)
        if constexpr (CKEY) atomicMax(&sh().ckey, key);     // the CTA's best key (see sens_hit)
        if (bst.gb) {  // prune mode: publish the score to the grid
            if (bst.thr > bst.pthr) atomicMax(bst.gb, s + 1u);
            bst.pthr = max(bst.pthr, bst.thr);
        }
    }
}

template <int W, int K, int SEL, int J>
__device__ __forceinline__ St<K> push(const Ctx<W> &c, const St<K> &st, uint32_t v) {
    St<K> s = st;
    const uint32_t vb = 1u << v;
    const uint4 t = sh().cm[v];
    if constexpr (SelT<SEL>::lin) {
        const uint32_t X = SelT<SEL>::useU ? st.U : st.bm[J];
        const int incv = SelT<SEL>::useU ? sh().inc[c.warp][v] : 0;
        s.acc = st.acc + SelT<SEL>::w12 * __popc(X) - incv + SelT<SEL>::w0 * __popc(t.x & X) + SelT<SEL>::w1 * __popc(t.y & X) +
                SelT<SEL>::w2 * __popc(t.z & X);
    } else {
        const uint32_t X = st.bm[J];
        s.acc = st.acc + __popc(t.x & X);
        s.acc2 = st.acc2 + __popc((t.y | t.z) & X);
    }
    s.U = st.U | vb;
    s.f[J] = v;
    const uint32_t fbJ = (uint32_t)(c.fb >> (8 * J)) & 0xFFu;
    const uint32_t fsJ = (uint32_t)(SelT<SEL>::canon ? c.fs >> (8 * J) : 0ull) & 0xFFu;
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
__device__ __forceinline__ void leaf_k1(const Ctx<W> &c, Best &bst) {
    const bool act = (c.F >> c.b) & 1u;
    const int s = (SelT<SEL>::lin) ? c.acc0 + c.leafC : 0;  // m = 0: census (0,0,0) has rank 0
    bst.cnt += act ? 1u : 0u;
    if (act && (uint32_t)s >= bst.bs) consider<W, 1>(c, bst, 1u << c.b, 0ull, (uint32_t)s);
}

// Level k-2 scan, dense over the W devices of the group.  Lane b writes its
// entry (increment of placing vertex k-2 on b, or a sentinel when b is not a
// candidate) into the group's table; then every lane (device of vertex k-1)
// ranks all W leaves (v, b) with its register column c.col (fully unrolled,
// compile-time indices) and keeps the max.  Within one scan a lane's leaves
// differ only in v, and among equal scores the smaller v is the lex-smaller
// device set (larger key), so the packed rank (score+1)*32 + (31-v) decides
// and the full key is built once, later.  Returns the max over v of
//   LIN:  tab[v] + col[v] (the rank minus `base`, added by the caller after
//         the threshold test, which keeps it off the dependency chain),
//         tab = 32 t2 | kNeg, col = T[v][b] + 31 - v
//   SENS: lut[base + tab[v] + col[v]] + 31 - v (the rank),  tab = t2 | kSent, col = D[v][b]
// The rank is < 32 when no leaf is valid.
// pack16 (single-query Eq. 2): the table holds 16-bit byte offsets and the
// lane's column holds two 16-bit offsets per register, so one LDS.128 brings 8
// table entries (broadcast loads cost 2 wavefronts each whatever their width)
// and one IADD3 forms two LUT addresses (every LUT byte offset is < 3*40*40*4
// < 2^16, so the halves never carry into each other).  (Measured against a
// u16 rank table with one IADD3 per leaf and VIADDMNMX.U16x2 over IMAD-packed
// pairs: 3 % slower, ALU-pipe bound.)
// lin16 (single-query Eq. 1 / 3, when the host proves the range fits): table
// entries and the lane's column are s16 pairs, two leaves per
// VIADDMNMX.S16x2 (see kNeg16T / kNeg16C).
template <int W, int SEL>
__device__ __forceinline__ int *tab_ptr(const Ctx<W> &c, int which) {
    int *t = sh().wl[c.warp].dense[which];
    if constexpr (SelT<SEL>::half) return reinterpret_cast<int *>(reinterpret_cast<uint16_t *>(t) + c.g * W);
    else return t + c.g * W;
}

template <int W, int SEL>
__device__ __forceinline__ void tab_put(const Ctx<W> &c, int *tab, int v) {
    if constexpr (SelT<SEL>::half) reinterpret_cast<uint16_t *>(tab)[c.b] = (uint16_t)v;
    else tab[c.b] = v;
}

// lin16 sentinels.  Valid table entries are 32 (t2 + ishift) in [0, 31135]
// (the host's lin16_fits), valid column entries 32 w + 31 - v in [0, 1631], so
// every valid leaf sums to [0, 32766].  An invalid table entry is -1632 and an
// invalid column entry -31136: any sum with a sentinel is negative and >= -32768
// (no s16 wrap).
constexpr int kNeg16T = -1632;
constexpr int kNeg16C = -31136;

template <int W, int SEL>
__device__ __forceinline__ int lin_entry(const Ctx<W> &c, bool ok, int t) {
    if constexpr (SelT<SEL>::lin16) return ok ? (t + c.ishift) * 32 : kNeg16T;
    else return ok ? t * 32 : kNeg;
}

template <int W, int SEL>
__device__ __forceinline__ int tab_entry(const Ctx<W> &c, uint32_t cand, int t2) {
    const bool mine = (cand >> c.b) & 1u;
    if constexpr (SelT<SEL>::lin) return lin_entry<W, SEL>(c, mine, t2);
    else return 4 * (mine ? t2 : c.xs * c.xs);  // byte offsets into the Eq. 2 table
}

template <int W, int SEL, bool TIE = true>
__device__ __forceinline__ int tab_scan(const Ctx<W> &c, const int *tab, int base) {
    if constexpr (SelT<SEL>::pack16 && !TIE) {
        // Hot scan of the single-query Eq. 2 kernels: the max LUT entry
        // (rank + 1) * 32 only, no tie-break -- per 2 leaves one IADD3, one SHF,
        // one IMAD (offset split), two gathers and one 3-input max.  The lane
        // with a hit (rank >= its best score, rare) rescans with TIE = true to
        // find the smallest v of that rank (sens_hit).  0 when no leaf is valid.
        const uint4 *t8 = reinterpret_cast<const uint4 *>(tab);
        const uint32_t b4 = __funnelshift_l(0u, (uint32_t)base, 2);
        const uint32_t bp = b4 | (b4 << 16);
        const int negk = c.negk;
        int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
        for (int q = 0; q < W / 8; ++q) {
            const uint4 e = t8[q];
            const uint32_t s0 = bp + e.x + (uint32_t)c.col[4 * q + 0];
            const uint32_t s1 = bp + e.y + (uint32_t)c.col[4 * q + 1];
            const uint32_t s2 = bp + e.z + (uint32_t)c.col[4 * q + 2];
            const uint32_t s3 = bp + e.w + (uint32_t)c.col[4 * q + 3];
            const int h0 = (int)(s0 >> 16), h1 = (int)(s1 >> 16), h2 = (int)(s2 >> 16), h3 = (int)(s3 >> 16);
            a0 = max(a0, max(lds_lut1((uint32_t)mad_lo(h0, negk, (int)s0)), lds_lut1((uint32_t)h0)));
            a1 = max(a1, max(lds_lut1((uint32_t)mad_lo(h1, negk, (int)s1)), lds_lut1((uint32_t)h1)));
            a2 = max(a2, max(lds_lut1((uint32_t)mad_lo(h2, negk, (int)s2)), lds_lut1((uint32_t)h2)));
            a3 = max(a3, max(lds_lut1((uint32_t)mad_lo(h3, negk, (int)s3)), lds_lut1((uint32_t)h3)));
        }
        return max(max(a0, a1), max(a2, a3));
    } else if constexpr (SelT<SEL>::pack16) {
        // Each register holds two 16-bit byte offsets; the high one is s >> 16
        // (ALU) and the low one s - (s >> 16) * 65536, an IMAD by a run-time
        // constant (FMA pipe), so the ALU pipe -- the binding one -- spends 3
        // ops per 2 leaves (IADD3, SHF, 3-input max); the (31 - v) tie-break
        // goes in as IMAD r*one + (31-v) (FMA pipe).
        const uint4 *t8 = reinterpret_cast<const uint4 *>(tab);
        const int *lut = lut1();
        const uint32_t b4 = __funnelshift_l(0u, (uint32_t)base, 2);
        const uint32_t bp = b4 | (b4 << 16);
        const int one = c.one, negk = c.negk;
        int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
        for (int q = 0; q < W / 8; ++q) {
            const uint4 e = t8[q];
            const uint32_t s0 = bp + e.x + (uint32_t)c.col[4 * q + 0];
            const uint32_t s1 = bp + e.y + (uint32_t)c.col[4 * q + 1];
            const uint32_t s2 = bp + e.z + (uint32_t)c.col[4 * q + 2];
            const uint32_t s3 = bp + e.w + (uint32_t)c.col[4 * q + 3];
            const int h0 = (int)(s0 >> 16), h1 = (int)(s1 >> 16), h2 = (int)(s2 >> 16), h3 = (int)(s3 >> 16);
            const int v = 8 * q;
            a0 = max(a0, max(lds_off(lut, (int)s0 + h0 * negk) * one + (31 - v), lds_off(lut, h0) * one + (30 - v)));
            a1 = max(a1, max(lds_off(lut, (int)s1 + h1 * negk) * one + (29 - v), lds_off(lut, h1) * one + (28 - v)));
            a2 = max(a2, max(lds_off(lut, (int)s2 + h2 * negk) * one + (27 - v), lds_off(lut, h2) * one + (26 - v)));
            a3 = max(a3, max(lds_off(lut, (int)s3 + h3 * negk) * one + (25 - v), lds_off(lut, h3) * one + (24 - v)));
        }
        return max(max(a0, a1), max(a2, a3));
    }
    if constexpr (SelT<SEL>::lin16) {
        // two leaves per VIADDMNMX.S16x2: table word q holds entries 2q / 2q+1,
        // column register q the lane's matching pair; four independent chains
        const uint4 *t8 = reinterpret_cast<const uint4 *>(tab);
        unsigned a0 = 0x80008000u, a1 = 0x80008000u, a2 = 0x80008000u, a3 = 0x80008000u;
#pragma unroll
        for (int q = 0; q < W / 8; ++q) {
            const uint4 e = t8[q];
            a0 = __viaddmax_s16x2(e.x, (unsigned)c.col[4 * q + 0], a0);
            a1 = __viaddmax_s16x2(e.y, (unsigned)c.col[4 * q + 1], a1);
            a2 = __viaddmax_s16x2(e.z, (unsigned)c.col[4 * q + 2], a2);
            a3 = __viaddmax_s16x2(e.w, (unsigned)c.col[4 * q + 3], a3);
        }
        const unsigned m2 = __vmaxs2(__vmaxs2(a0, a1), __vmaxs2(a2, a3));
        const int r = max((int)(short)(m2 & 0xFFFFu), (int)m2 >> 16);
        return r < 0 ? kNeg : r;  // no valid leaf
    }
    const int4 *t4 = reinterpret_cast<const int4 *>(tab);
    int best = 0;
    // Pipe balance: the integer ALU pipe (add-max, 3-input max, address adds)
    // and the FMA pipe (IMAD) each retire a warp instruction every 2 cycles.
    // A fused add-max costs one ALU slot per leaf; an add done as IMAD x*one+y
    // (c.one = 1 at run time, so the compiler keeps the IMAD) followed by a
    // 3-input max over two leaves costs one FMA slot + half an ALU slot.
    if constexpr (SelT<SEL>::lin) {
        // four independent fused add-max chains (VIADDMNMX); measured faster
        // than moving part of the adds to the FMA pipe (the loop is latency-,
        // not pipe-bound at 4 warps per scheduler)
        const int4 e0 = t4[0];
        int b0 = e0.x + c.col[0], b1 = e0.y + c.col[1], b2 = e0.z + c.col[2], b3 = e0.w + c.col[3];
#pragma unroll
        for (int q = 1; q < W / 4; ++q) {
            const int4 e = t4[q];
            b0 = max(b0, e.x + c.col[4 * q + 0]);
            b1 = max(b1, e.y + c.col[4 * q + 1]);
            b2 = max(b2, e.z + c.col[4 * q + 2]);
            b3 = max(b3, e.w + c.col[4 * q + 3]);
        }
        best = max(max(b0, b1), max(b2, b3));
    } else {
        // table, column and base are byte offsets into the Eq. 2 table: one
        // IADD3 per leaf gives the address.  4*base goes through a funnel shift
        // so that the compiler does not re-split the sum into a multiply-add
        // per leaf.
        const int *lb = reinterpret_cast<const int *>(reinterpret_cast<const char *>(sh_lut() + c.lut) +
                                                      (int)__funnelshift_l(0u, (uint32_t)base, 2));
        // the (31 - v) tie-break goes in as IMAD r*one + (31-v), two leaves per 3-input max
        int b0 = 0, b1 = 0;
        const int one = c.one;
#pragma unroll
        for (int q = 0; q < W / 4; ++q) {
            const int4 e = t4[q];
            const int r0 = lds_off(lb, e.x + c.col[4 * q + 0]) * one + (31 - (4 * q + 0));
            const int r1 = lds_off(lb, e.y + c.col[4 * q + 1]) * one + (31 - (4 * q + 1));
            const int r2 = lds_off(lb, e.z + c.col[4 * q + 2]) * one + (31 - (4 * q + 2));
            const int r3 = lds_off(lb, e.w + c.col[4 * q + 3]) * one + (31 - (4 * q + 3));
            b0 = max(b0, max(r0, r1));
            b1 = max(b1, max(r2, r3));
        }
        best = max(b0, b1);
    }
    return best;
}

// lin16 hot scan against the lane's threshold t (= thr - off): the four s16x2
// chains start at clamp(t - 1, -1, 32766) in both halves, so the scan has a
// hit iff their max differs from that start (valid leaf sums are >= 0, invalid
// ones < 0, none above 32766); only a hit unpacks the halves (s16_best).
// Returns the s16x2 max; `i0` gets the start value.
template <int W, int SEL>
__device__ __forceinline__ unsigned tab_scan_thr(const Ctx<W> &c, const int *tab, int t, unsigned &i0) {
    static_assert(SelT<SEL>::lin16, "lin16 only");
    const uint4 *t8 = reinterpret_cast<const uint4 *>(tab);
    const int t0 = min(max(t - 1, -1), 32766);
    i0 = __byte_perm((unsigned)t0, 0u, 0x1010);
    unsigned a0 = i0, a1 = i0, a2 = i0, a3 = i0;
#pragma unroll
    for (int q = 0; q < W / 8; ++q) {
        const uint4 e = t8[q];
        a0 = __viaddmax_s16x2(e.x, (unsigned)c.col[4 * q + 0], a0);
        a1 = __viaddmax_s16x2(e.y, (unsigned)c.col[4 * q + 1], a1);
        a2 = __viaddmax_s16x2(e.z, (unsigned)c.col[4 * q + 2], a2);
        a3 = __viaddmax_s16x2(e.w, (unsigned)c.col[4 * q + 3], a3);
    }
    return __vmaxs2(__vmaxs2(a0, a1), __vmaxs2(a2, a3));
}

__device__ __forceinline__ int s16_best(unsigned m2) { return max((int)(short)(m2 & 0xFFFFu), (int)m2 >> 16); }

// ---------------------------------------------------------------- static-table scans (SelT::stat)
// lin16: as tab_scan_thr, the leaf pair sums being row[q] + colT[q] (s16x2)
template <int W>
__device__ __forceinline__ unsigned scan_row_thr(uint32_t row, const uint32_t (&colT)[W / 2], int t,
                                                 unsigned &i0) {
    const int t0 = min(max(t - 1, -1), 32766);
    i0 = __byte_perm((unsigned)t0, 0u, 0x1010);
    unsigned a0 = i0, a1 = i0, a2 = i0, a3 = i0;
#pragma unroll
    for (int q = 0; q < W / 8; ++q) {
        const uint4 e = lds_row<false>(row + 16u * q);
        a0 = __viaddmax_s16x2(e.x, colT[4 * q + 0], a0);
        a1 = __viaddmax_s16x2(e.y, colT[4 * q + 1], a1);
        a2 = __viaddmax_s16x2(e.z, colT[4 * q + 2], a2);
        a3 = __viaddmax_s16x2(e.w, colT[4 * q + 3], a3);
    }
    return __vmaxs2(__vmaxs2(a0, a1), __vmaxs2(a2, a3));
}

// Eq. 2: max LUT entry over the leaves, byte offsets bp + row[q] + colT[q]
// (the pack16 scan of tab_scan<.., false>)
template <int W>
__device__ __forceinline__ int scan_row_max(uint32_t row, const uint32_t (&colT)[W / 2], int base, int negk) {
    const uint32_t b4 = __funnelshift_l(0u, (uint32_t)base, 2);
    const uint32_t bp = b4 | (b4 << 16);
    int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int q = 0; q < W / 8; ++q) {
        const uint4 e = lds_row<true>(row + 16u * q);
        const uint32_t s0 = bp + e.x + colT[4 * q + 0];
        const uint32_t s1 = bp + e.y + colT[4 * q + 1];
        const uint32_t s2 = bp + e.z + colT[4 * q + 2];
        const uint32_t s3 = bp + e.w + colT[4 * q + 3];
        const int h0 = (int)(s0 >> 16), h1 = (int)(s1 >> 16), h2 = (int)(s2 >> 16), h3 = (int)(s3 >> 16);
        a0 = max(a0, max(lds_lut1((uint32_t)mad_lo(h0, negk, (int)s0)), lds_lut1((uint32_t)h0)));
        a1 = max(a1, max(lds_lut1((uint32_t)mad_lo(h1, negk, (int)s1)), lds_lut1((uint32_t)h1)));
        a2 = max(a2, max(lds_lut1((uint32_t)mad_lo(h2, negk, (int)s2)), lds_lut1((uint32_t)h2)));
        a3 = max(a3, max(lds_lut1((uint32_t)mad_lo(h3, negk, (int)s3)), lds_lut1((uint32_t)h3)));
    }
    return max(max(a0, a1), max(a2, a3));
}

// Eq. 2 rescan of a hit: the packed rank (rank + 1) * 32 + 31 - v
template <int W>
__device__ __forceinline__ int scan_row_tie(uint32_t row, const uint32_t (&colT)[W / 2], int base, int one,
                                            int negk) {
    const int *lut = lut1();
    const uint32_t b4 = __funnelshift_l(0u, (uint32_t)base, 2);
    const uint32_t bp = b4 | (b4 << 16);
    int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int q = 0; q < W / 8; ++q) {
        const uint4 e = lds_row<true>(row + 16u * q);
        const uint32_t s0 = bp + e.x + colT[4 * q + 0];
        const uint32_t s1 = bp + e.y + colT[4 * q + 1];
        const uint32_t s2 = bp + e.z + colT[4 * q + 2];
        const uint32_t s3 = bp + e.w + colT[4 * q + 3];
        const int h0 = (int)(s0 >> 16), h1 = (int)(s1 >> 16), h2 = (int)(s2 >> 16), h3 = (int)(s3 >> 16);
        const int v = 8 * q;
        a0 = max(a0, max(lds_off(lut, (int)s0 + h0 * negk) * one + (31 - v), lds_off(lut, h0) * one + (30 - v)));
        a1 = max(a1, max(lds_off(lut, (int)s1 + h1 * negk) * one + (29 - v), lds_off(lut, h1) * one + (28 - v)));
        a2 = max(a2, max(lds_off(lut, (int)s2 + h2 * negk) * one + (27 - v), lds_off(lut, h2) * one + (26 - v)));
        a3 = max(a3, max(lds_off(lut, (int)s3 + h3 * negk) * one + (25 - v), lds_off(lut, h3) * one + (24 - v)));
    }
    return max(max(a0, a1), max(a2, a3));
}

template <int W, int SEL>
__device__ __forceinline__ int scan_dense(const Ctx<W> &c, uint32_t cand, int t2, int base) {
    int *tab = tab_ptr<W, SEL>(c, 0);
    __syncwarp(c.gmask);  // previous readers of the table are done
    tab_put<W, SEL>(c, tab, tab_entry<W, SEL>(c, cand, t2));
    __syncwarp(c.gmask);
    return tab_scan<W, SEL, !SelT<SEL>::pack16>(c, tab, base);
}

// pack16 hit (scan max `raw` = (rank + 1) * 32 >= the lane's threshold): the
// packed rank with the (31 - v) tie-break, or -1 when the hit cannot change
// the result.  Hits are frequent (Eq. 2 ranks saturate: ~40 % of the C4 scans
// reach the lane's best score), so they are filtered against the CTA's best
// key (Shared::ckey, raised by every lane's improvement) before the rescan:
// a leaf of this scan has score s = raw / 32 - 1 and a device set no smaller
// than Ufix + the smallest valid v (`vm` = the lane's valid v), so if
// (s, that set) does not beat the CTA key's (score, set) no leaf of the scan
// can win anywhere (the final result is a max).  The lane's threshold is
// raised to the CTA's score on the way.
template <int W>
__device__ __forceinline__ bool sens_may_win(const Ctx<W> &c, Best &bst, int raw, uint32_t Ufix, uint32_t vm) {
    const unsigned long long chi = *reinterpret_cast<volatile unsigned long long *>(&sh().ckey) >> c.eb;
    bst.thr = max(bst.thr, ((int)(uint32_t)(chi >> W) + 1) * 32);
    if (raw < bst.thr) return false;
    const uint32_t sbmax = __brev(Ufix | (vm & (0u - vm))) >> (32 - W);
    const unsigned long long hi = ((unsigned long long)((uint32_t)raw >> 5) - 1ull) << W | sbmax;
    return !(hi < chi || (hi == chi && c.clique));
}

template <int W, int SEL>
__device__ __forceinline__ int sens_hit(const Ctx<W> &c, Best &bst, int raw, uint32_t Ufix, uint32_t vm, int base) {
    if (!sens_may_win<W>(c, bst, raw, Ufix, vm)) return -1;
    return tab_scan<W, SEL, true>(c, tab_ptr<W, SEL>(c, 0), base);
}

template <int W>
__device__ __forceinline__ int grp_max(const Ctx<W> &c, int x) {
    if constexpr (W == 32) {
        return __reduce_max_sync(kFull, x);
    } else {
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(c.gmask, x, o, W));
        return x;
    }
}

// Prune mode: does the k-2 scan with this lane's table entry / base have a leaf
// that can still matter anywhere in the grid?  Upper bound of the lane's
// packed ranks: additive scores max_v tab[v] + max_v col[v] + base; Eq. 2 the
// precomputed max rank reachable from the lane's census by the edges the scan
// adds (`ubtab`).  Group-uniform result.
template <int W, int SEL>
__device__ __forceinline__ bool scan_needed(const Ctx<W> &c, const Best &bst, int entry, int base, bool laneok) {
    int ub;
    if constexpr (SelT<SEL>::lin) ub = base + grp_max<W>(c, entry) + c.colmax;
    else ub = lut1()[3 * c.xs * c.xs + base] + 31;  // prune mode: single-query only
    return __any_sync(c.gmask, laneok && ub >= bst.pthr);
}

// The two innermost levels: vertex k-2 walks the devices of `cand`, vertex
// k-1 sits on the lanes.  Vertices 0..k-3 are placed.
template <int W, int K, int SEL>
__device__ __forceinline__ void inner(const Ctx<W> &c, const St<K> &st, uint32_t cand, Best &bst) {
    constexpr int J = K - 2;
    const uint32_t b = (uint32_t)c.b;
    const uint32_t fbJ = (uint32_t)(c.fb >> (8 * J)) & 0xFFu;
    const uint32_t fsJ = (uint32_t)(SelT<SEL>::canon ? c.fs >> (8 * J) : 0ull) & 0xFFu;
    const bool eK = (fbJ >> (K - 1)) & 1u;   // pattern edge (k-2, k-1)
    const bool dep = (fsJ >> (K - 1)) & 1u;  // lex-leader f(k-2) < f(k-1)
    int t2, base;
    if constexpr (SelT<SEL>::lin) {
        const uint32_t X2 = SelT<SEL>::useU ? st.U : st.bm[J];
        const uint32_t X1 = SelT<SEL>::useU ? st.U : st.bm[K - 1];
        t2 = SelT<SEL>::w12 * __popc(X2) - (SelT<SEL>::useU ? c.incb : 0) + SelT<SEL>::w0 * __popc(c.cm0 & X2) + SelT<SEL>::w1 * __popc(c.cm1 & X2) +
             SelT<SEL>::w2 * __popc(c.cm2 & X2);
        const int lp = c.laneC + SelT<SEL>::w12 * __popc(X1) + SelT<SEL>::w0 * __popc(c.cm0 & X1) + SelT<SEL>::w1 * __popc(c.cm1 & X1) +
                       SelT<SEL>::w2 * __popc(c.cm2 & X1);
        base = (st.acc + lp + 1 - c.ishift) * 32;
    } else {
        const uint32_t X2 = st.bm[J], X1 = st.bm[K - 1];
        t2 = __popc(c.cm0 & X2) * c.xs + __popc(c.cm12 & X2);
        base = (st.acc + __popc(c.cm0 & X1)) * c.xs + st.acc2 + __popc(c.cm12 & X1);  // census index
    }
    const bool laneok = ((c.F & ~st.U & alw<SEL>(st.al[K - 1])) >> b) & 1u;
    // leaves counted: v in cand with v != b (and v < b if canonical-ordered)
    const uint32_t M = laneok ? (dep ? ((1u << b) - 1u) : ~(1u << b)) : 0u;
    bst.cnt += (uint32_t)__popc(M & cand);
    const int off = SelT<SEL>::lin ? base : 0;
    // a leaf below the CTA's best score cannot win anywhere (max is global)
    if constexpr (SelT<SEL>::cta) bst.thr = max(bst.thr, sh().cthr);
    const int thr = bst.thr - off;
    int raw = scan_dense<W, SEL>(c, cand, t2, base);
    if (laneok && raw >= thr) {  // rank >= 32 and its score >= the lane's best score
        if constexpr (SelT<SEL>::pack16) {
            raw = sens_hit<W, SEL>(c, bst, raw, st.U | (1u << b), M & cand, base);
            if (raw < 0) return;
        }
        const int best = raw + off;
        const uint32_t s = (uint32_t)(best >> 5) - 1u;
        {
            const uint32_t bestv = 31u - (uint32_t)(best & 31);
            unsigned long long fpack = pack_f<K>(st);
            fpack |= (unsigned long long)bestv << (8 * J);
            consider<W, K, SelT<SEL>::cta, SelT<SEL>::pack16>(c, bst, st.U | (1u << bestv) | (1u << b), fpack, s);
        }
    }
}

// The three innermost levels: vertex k-3 walks `cand3` (uniform loop over a
// per-group list of (v3, increment of placing k-3 on v3) built lane-parallel);
// for every v3 the lane values are updated by ONE table lookup (w(v3,b) or the
// census delta) and the k-2 list scan runs.  Vertices 0..k-4 are placed.
template <int W, int K, int SEL>
__device__ __forceinline__ void inner3(const Ctx<W> &c, const St<K> &st, uint32_t cand3, Best &bst) {
    constexpr int J3 = K - 3, J2 = K - 2, J1 = K - 1;
    const uint32_t b = (uint32_t)c.b;
    const uint32_t fb3 = (uint32_t)(c.fb >> (8 * J3)) & 0xFFu, fs3 = (uint32_t)(SelT<SEL>::canon ? c.fs >> (8 * J3) : 0ull) & 0xFFu;
    const uint32_t fb2 = (uint32_t)(c.fb >> (8 * J2)) & 0xFFu, fs2 = (uint32_t)(SelT<SEL>::canon ? c.fs >> (8 * J2) : 0ull) & 0xFFu;
    const bool e32 = (fb3 >> J2) & 1u, e31 = (fb3 >> J1) & 1u, e21 = (fb2 >> J1) & 1u;
    const bool d32 = (fs3 >> J2) & 1u, d31 = (fs3 >> J1) & 1u, d21 = (fs2 >> J1) & 1u;
    // lane values over the placed vertices 0..k-4:
    //   t3 = increment of placing k-3 on b, t2b = of placing k-2 on b,
    //   lpb = leaf partial of k-1 on b; v3 then adds m32 w3, m31 w3.
    int t3, t2b, lpb, m32, m31, A;
    const int *wcol;
    if constexpr (SelT<SEL>::lin) {
        const uint32_t X3 = SelT<SEL>::useU ? st.U : st.bm[J3];
        const uint32_t X2 = SelT<SEL>::useU ? st.U : st.bm[J2];
        const uint32_t X1 = SelT<SEL>::useU ? st.U : st.bm[J1];
        const int inc = SelT<SEL>::useU ? c.incb : 0;
        t3 = SelT<SEL>::w12 * __popc(X3) - inc + SelT<SEL>::w0 * __popc(c.cm0 & X3) + SelT<SEL>::w1 * __popc(c.cm1 & X3) +
             SelT<SEL>::w2 * __popc(c.cm2 & X3);
        t2b = SelT<SEL>::w12 * __popc(X2) - inc + SelT<SEL>::w0 * __popc(c.cm0 & X2) + SelT<SEL>::w1 * __popc(c.cm1 & X2) +
              SelT<SEL>::w2 * __popc(c.cm2 & X2);
        lpb = c.laneC + SelT<SEL>::w12 * __popc(X1) + SelT<SEL>::w0 * __popc(c.cm0 & X1) + SelT<SEL>::w1 * __popc(c.cm1 & X1) +
              SelT<SEL>::w2 * __popc(c.cm2 & X1);
        m32 = (SelT<SEL>::w12 != 0 && (SelT<SEL>::useU || e32)) ? 1 : 0;
        m31 = (SelT<SEL>::w12 != 0 && (SelT<SEL>::useU || e31)) ? 1 : 0;
        A = st.acc;
        wcol = sh().twp + b;
    } else {
        const uint32_t X3 = st.bm[J3], X2 = st.bm[J2], X1 = st.bm[J1];
        t3 = __popc(c.cm0 & X3) * c.xs + __popc(c.cm12 & X3);
        t2b = __popc(c.cm0 & X2) * c.xs + __popc(c.cm12 & X2);
        lpb = __popc(c.cm0 & X1) * c.xs + __popc(c.cm12 & X1);
        m32 = e32 ? 1 : 0;
        m31 = e31 ? 1 : 0;
        A = st.acc * c.xs + st.acc2;
        wcol = sh().tdl + b;
    }
    int2 *L3 = sh().wl[c.warp].l3 + c.g * W;
    const uint32_t n3 = (uint32_t)__popc(cand3);
    __syncwarp(c.gmask);  // previous readers of the k-3 list are done
    if ((cand3 >> b) & 1u) L3[__popc(cand3 & ((1u << b) - 1u))] = make_int2((int)b, t3);
    __syncwarp(c.gmask);
    const bool okb = ((c.F & ~st.U & alw<SEL>(st.al[J1])) >> b) & 1u;
    const uint32_t cand2b = c.F & ~st.U & alw<SEL>(st.al[J2]);
    const unsigned long long fbase = pack_f<K>(st);
    const bool dep = d32 || d31 || d21 || SelT<SEL>::prune;  // prune mode counts the scans it runs
    // Hit threshold: a leaf matters only if its score reaches both the lane's
    // best and the best any lane of this CTA has found (a lower score loses
    // to that key in the final max; ties still reach the key builder for the
    // tie-break).  Sharing the CTA's best keeps most lanes out of the
    // divergent key-building path early in the search.
    // (a lower score loses to the CTA's best key in the final max, so the
    // lane's threshold may be raised to it; ties still reach the key builder)
    if constexpr (SelT<SEL>::cta) bst.thr = max(bst.thr, sh().cthr);
    if constexpr (SelT<SEL>::prune) {
        const unsigned g = ld_relaxed(bst.gb);
        bst.pthr = max(bst.pthr, (int)(g * 32u));
        if constexpr (SelT<SEL>::lin) {
            // Bound of the whole prefix subtree for this lane (vertex k-1 on b).
            // A leaf (v3, v) ranks 32 (A + lpb + 1 + t3(v3) + m31 w(v3,b)
            // + t2b(v) + m32 w(v3,v)) + col_b[v]; bound the v3 part and the v
            // part separately with two dense scans (tables 32 t3 and 32 t2b
            // over the candidates, the lane's column; col_b >= 32 w(., b)
            // when the edge (k-2, k-1) exists, else the v3 edge takes the
            // largest weight) and w(v3, v) by 50.
            int *ta = tab_ptr<W, SEL>(c, 0), *tb2 = tab_ptr<W, SEL>(c, 1);
            __syncwarp(c.gmask);
            tab_put<W, SEL>(c, ta, lin_entry<W, SEL>(c, (cand3 >> b) & 1u, t3));
            tab_put<W, SEL>(c, tb2, lin_entry<W, SEL>(c, (cand2b >> b) & 1u, t2b));
            __syncwarp(c.gmask);
            // the column carries the (., b) weights unless the edge (k-2, k-1) is
            // absent (Eq. 1), and has no order sentinels unless f(k-2) < f(k-1)
            // is a lex-leader constraint
            const bool colw = (SelT<SEL>::useU || e21) && !d21;
            const int s3 = colw ? tab_scan<W, SEL>(c, ta, 0) : 32 * grp_max<W>(c, ((cand3 >> b) & 1u) ? t3 : kNeg) +
                                                            32 * 50 * SelT<SEL>::wt * m31;
            const int s2 = tab_scan<W, SEL>(c, tb2, 0);
            // lin16: the scanned entries carry + 32 ishift each
            const int ub = 32 * (A + lpb + 1 + m32 * 50 * SelT<SEL>::wt) + s3 + s2 - (colw ? 64 : 32) * c.ishift;
            if (!__any_sync(c.gmask, okb && ub >= bst.pthr)) return;
        }
    }
    if (!dep && okb) {
        // leaves of this lane: every (v3, v) with v3 in cand3, v in cand2b, v3, v, b distinct
        const uint32_t nb = ~(1u << b);
        bst.cnt += (uint32_t)(__popc(cand3 & nb) * __popc(cand2b & nb) - __popc(cand3 & cand2b & nb));
    }
    if constexpr (!SelT<SEL>::lin) {
        // Eq. 2: one v3 per iteration (the scan is shared-memory bound; pairing
        // measured slower)
        for (uint32_t i = 0; i < n3; ++i) {
            const int2 e3 = L3[i];
            const uint32_t v3 = (uint32_t)e3.x;
            const int w3 = wcol[v3 * 32];
            const uint32_t cand2 = cand2b & ~(1u << v3) & (d32 ? (0xFFFFFFFEu << v3) : kFull);
            const bool laneok = okb && b != v3 && (!d31 || b > v3);
            const int base = A + e3.y + lpb + m31 * w3;
            if constexpr (SelT<SEL>::prune) {
                if (!scan_needed<W, SEL>(c, bst, 0, base, laneok)) continue;
            }
            if (dep) {
                const uint32_t M = laneok ? (d21 ? ((1u << b) - 1u) : ~(1u << b)) : 0u;
                bst.cnt += (uint32_t)__popc(M & cand2);
            }
            int raw = scan_dense<W, SEL>(c, cand2, t2b + m32 * w3, base);
            if (laneok && raw >= bst.thr) {  // rank >= 32 and its score >= the lane's best score
                if constexpr (SelT<SEL>::pack16) {
                    const uint32_t vm = cand2 & (d21 ? ((1u << b) - 1u) : ~(1u << b));
                    raw = sens_hit<W, SEL>(c, bst, raw, st.U | (1u << v3) | (1u << b), vm, base);
                    if (raw < 0) continue;
                }
                const uint32_t bestv = 31u - (uint32_t)(raw & 31);
                const unsigned long long fpack =
                    fbase | ((unsigned long long)v3 << (8 * J3)) | ((unsigned long long)bestv << (8 * J2));
                consider<W, K, SelT<SEL>::cta, SelT<SEL>::pack16>(c, bst, st.U | (1u << v3) | (1u << bestv) | (1u << b), fpack,
                               (uint32_t)(raw >> 5) - 1u);
            }
        }
        return;
    }
    // two v3 per iteration (tables A and B): twice the independent work
    // between the warp syncs and one threshold branch for both scans
    int *tabA = tab_ptr<W, SEL>(c, 0);
    int *tabB = tab_ptr<W, SEL>(c, 1);
    for (uint32_t i = 0; i < n3; i += 2) {
        const bool hasB = i + 1 < n3;
        const int2 eA = L3[i], eB = L3[hasB ? i + 1 : i];
        const uint32_t vA = (uint32_t)eA.x, vB = (uint32_t)eB.x;
        const int wA = wcol[vA * 32], wB = wcol[vB * 32];
        const uint32_t cA = cand2b & ~(1u << vA) & (d32 ? (0xFFFFFFFEu << vA) : kFull);
        const uint32_t cB = cand2b & ~(1u << vB) & (d32 ? (0xFFFFFFFEu << vB) : kFull);
        bool okA = okb && b != vA && (!d31 || b > vA);
        bool okB = hasB && okb && b != vB && (!d31 || b > vB);
        const int lpA = lpb + m31 * wA, lpB = lpb + m31 * wB;
        const int baseA = (SelT<SEL>::lin) ? (A + eA.y + lpA + 1 - c.ishift) * 32 : A + eA.y + lpA;
        const int baseB = (SelT<SEL>::lin) ? (A + eB.y + lpB + 1 - c.ishift) * 32 : A + eB.y + lpB;
        const int offA = SelT<SEL>::lin ? baseA : 0, offB = SelT<SEL>::lin ? baseB : 0;
        const int entA = tab_entry<W, SEL>(c, cA, t2b + m32 * wA);
        const int entB = tab_entry<W, SEL>(c, cB, t2b + m32 * wB);
        bool runA = true, runB = true;
        if constexpr (SelT<SEL>::prune) {
            runA = scan_needed<W, SEL>(c, bst, entA, baseA, okA);
            runB = scan_needed<W, SEL>(c, bst, entB, baseB, okB);
            if (!runA && !runB) continue;
            okA = okA && runA;  // a skipped scan counts no leaves and proposes none
            okB = okB && runB;
        }
        if (dep) {
            const uint32_t M = d21 ? ((1u << b) - 1u) : ~(1u << b);
            bst.cnt += (uint32_t)(okA ? __popc(M & cA) : 0) + (uint32_t)(okB ? __popc(M & cB) : 0);
        }
        __syncwarp(c.gmask);  // previous readers of the tables are done
        tab_put<W, SEL>(c, tabA, entA);
        tab_put<W, SEL>(c, tabB, entB);
        __syncwarp(c.gmask);
        int rawA, rawB;
        bool hitA, hitB;
        unsigned mA = 0, mB = 0;
        if constexpr (SelT<SEL>::lin16) {
            unsigned iA = 0, iB = 0;
            if (runA) mA = tab_scan_thr<W, SEL>(c, tabA, bst.thr - offA, iA);
            if (runB) mB = tab_scan_thr<W, SEL>(c, tabB, bst.thr - offB, iB);
            hitA = okA && runA && mA != iA;
            hitB = okB && runB && mB != iB;
        } else {
            rawA = runA ? tab_scan<W, SEL>(c, tabA, baseA) : kNeg;
            rawB = runB ? tab_scan<W, SEL>(c, tabB, baseB) : kNeg;
            hitA = okA && rawA >= bst.thr - offA;
            hitB = okB && rawB >= bst.thr - offB;
        }
        if (hitA || hitB) {  // a rank >= 32 whose score >= the lane's / CTA's best score
            if constexpr (SelT<SEL>::lin16) {
                rawA = s16_best(mA);
                rawB = s16_best(mB);
            }
            if (hitA) {
                const int best = rawA + offA;
                const uint32_t bestv = 31u - (uint32_t)(best & 31);
                const unsigned long long fpack =
                    fbase | ((unsigned long long)vA << (8 * J3)) | ((unsigned long long)bestv << (8 * J2));
                consider<W, K, SelT<SEL>::cta, SelT<SEL>::pack16>(c, bst, st.U | (1u << vA) | (1u << bestv) | (1u << b), fpack,
                               (uint32_t)(best >> 5) - 1u);
            }
            if (hitB && rawB >= bst.thr - offB) {
                const int best = rawB + offB;
                const uint32_t bestv = 31u - (uint32_t)(best & 31);
                const unsigned long long fpack =
                    fbase | ((unsigned long long)vB << (8 * J3)) | ((unsigned long long)bestv << (8 * J2));
                consider<W, K, SelT<SEL>::cta, SelT<SEL>::pack16>(c, bst, st.U | (1u << vB) | (1u << bestv) | (1u << b), fpack,
                               (uint32_t)(best >> 5) - 1u);
            }
        }
    }
}

// ---------------------------------------------------------------- static-table inner levels
// The lane's column re-based on this prefix: colT[q] = column pair q + the
// pair (2q, 2q+1) of the lanes' T2 entries (`entry` = this lane's entry as the
// device of vertex k-2).  The caller has synced the group since the last
// reader of dense[0]; this syncs after the write.
template <int W, int SEL>
__device__ __forceinline__ void stat_col(const Ctx<W> &c, int entry, uint32_t (&colT)[W / 2]) {
    uint16_t *t = reinterpret_cast<uint16_t *>(sh().wl[c.warp].dense[0]) + c.g * W;
    t[c.b] = (uint16_t)entry;
    __syncwarp(c.gmask);
    const uint4 *t8 = reinterpret_cast<const uint4 *>(t);
    const uint32_t *cs = stt<SelT<SEL>::pack16>().col + c.b;
#pragma unroll
    for (int q = 0; q < W / 8; ++q) {
        const uint4 e = t8[q];
        const uint32_t ev[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t cv = cs[(4 * q + j) * W];
            if constexpr (SelT<SEL>::lin16) colT[4 * q + j] = __viaddmax_s16x2(cv, ev[j], 0x80008000u);  // s16x2 add
            else colT[4 * q + j] = cv + ev[j];  // byte offsets, no carry between the halves
        }
    }
}

// T2 entry of this lane as the device of vertex k-2 (`ok`: a candidate)
template <int W, int SEL>
__device__ __forceinline__ int stat_entry(const Ctx<W> &c, bool ok, int t2) {
    if constexpr (SelT<SEL>::lin16) return ok ? (t2 + c.ishift) * 32 : kStX;
    else return 4 * (ok ? t2 : c.xs * c.xs);
}

// inner() on the static tables: the k-2 scan reads the all-zero row W.
template <int W, int K, int SEL>
__device__ __forceinline__ void inners(const Ctx<W> &c, const St<K> &st, uint32_t cand, Best &bst) {
    constexpr int J = K - 2;
    const uint32_t b = (uint32_t)c.b;
    const uint32_t fsJ = (uint32_t)(SelT<SEL>::canon ? c.fs >> (8 * J) : 0ull) & 0xFFu;
    const bool dep = (fsJ >> (K - 1)) & 1u;  // lex-leader f(k-2) < f(k-1)
    int t2, base;
    if constexpr (SelT<SEL>::lin) {
        const uint32_t X2 = SelT<SEL>::useU ? st.U : st.bm[J];
        const uint32_t X1 = SelT<SEL>::useU ? st.U : st.bm[K - 1];
        t2 = SelT<SEL>::w12 * __popc(X2) - (SelT<SEL>::useU ? c.incb : 0) + SelT<SEL>::w0 * __popc(c.cm0 & X2) +
             SelT<SEL>::w1 * __popc(c.cm1 & X2) + SelT<SEL>::w2 * __popc(c.cm2 & X2);
        const int lp = c.laneC + SelT<SEL>::w12 * __popc(X1) + SelT<SEL>::w0 * __popc(c.cm0 & X1) +
                       SelT<SEL>::w1 * __popc(c.cm1 & X1) + SelT<SEL>::w2 * __popc(c.cm2 & X1);
        base = (st.acc + lp + 1 - c.ishift) * 32;
    } else {
        const uint32_t X2 = st.bm[J], X1 = st.bm[K - 1];
        t2 = __popc(c.cm0 & X2) * c.xs + __popc(c.cm12 & X2);
        base = (st.acc + __popc(c.cm0 & X1)) * c.xs + st.acc2 + __popc(c.cm12 & X1);  // census index
    }
    const bool laneok = ((c.F & ~st.U & alw<SEL>(st.al[K - 1])) >> b) & 1u;
    const uint32_t M = laneok ? (dep ? ((1u << b) - 1u) : ~(1u << b)) : 0u;
    bst.cnt += (uint32_t)__popc(M & cand);
    if constexpr (SelT<SEL>::cta) bst.thr = max(bst.thr, sh().cthr);
    uint32_t colT[W / 2];
    __syncwarp(c.gmask);  // previous readers of dense[0] are done
    stat_col<W, SEL>(c, stat_entry<W, SEL>(c, (cand >> b) & 1u, t2), colT);
    const uint32_t row = 4u * W * (W / 2);  // byte offset of row W
    int raw;
    if constexpr (SelT<SEL>::lin16) {
        unsigned i0;
        const unsigned m2 = scan_row_thr<W>(row, colT, bst.thr - base, i0);
        if (!(laneok && m2 != i0)) return;
        raw = s16_best(m2) + base;
    } else {
        raw = scan_row_max<W>(row, colT, base, c.negk);
        if (!(laneok && raw >= bst.thr)) return;
        if (!sens_may_win<W>(c, bst, raw, st.U | (1u << b), M & cand)) return;
        raw = scan_row_tie<W>(row, colT, base, c.one, c.negk);
    }
    const uint32_t bestv = 31u - (uint32_t)(raw & 31);
    const unsigned long long fpack = pack_f<K>(st) | ((unsigned long long)bestv << (8 * J));
    consider<W, K, SelT<SEL>::cta, SelT<SEL>::pack16>(c, bst, st.U | (1u << bestv) | (1u << b), fpack,
                                                      (uint32_t)(raw >> 5) - 1u);
}

// inner3() on the static tables (see SelT::stat): per v3 no table is built and
// no warp sync runs; the scan reads row v3 and the prefix-based column colT.
template <int W, int K, int SEL>
__device__ __forceinline__ void inner3s(const Ctx<W> &c, const St<K> &st, uint32_t cand3, Best &bst) {
    constexpr int J3 = K - 3, J2 = K - 2, J1 = K - 1;
    const uint32_t b = (uint32_t)c.b;
    const uint32_t fs3 = (uint32_t)(SelT<SEL>::canon ? c.fs >> (8 * J3) : 0ull) & 0xFFu;
    const uint32_t fb3 = (uint32_t)(c.fb >> (8 * J3)) & 0xFFu;
    const uint32_t fs2 = (uint32_t)(SelT<SEL>::canon ? c.fs >> (8 * J2) : 0ull) & 0xFFu;
    const bool e31 = (fb3 >> J1) & 1u;
    const bool d32 = (fs3 >> J2) & 1u, d31 = (fs3 >> J1) & 1u, d21 = (fs2 >> J1) & 1u;
    // lane values over the placed vertices 0..k-4 (see inner3); the (k-3, k-2)
    // edge term lives in the static row, the (k-3, k-1) term is m31 w3
    int t3, t2b, lpb, m31, A;
    const int *wcol;
    if constexpr (SelT<SEL>::lin) {
        const uint32_t X3 = SelT<SEL>::useU ? st.U : st.bm[J3];
        const uint32_t X2 = SelT<SEL>::useU ? st.U : st.bm[J2];
        const uint32_t X1 = SelT<SEL>::useU ? st.U : st.bm[J1];
        const int inc = SelT<SEL>::useU ? c.incb : 0;
        t3 = SelT<SEL>::w12 * __popc(X3) - inc + SelT<SEL>::w0 * __popc(c.cm0 & X3) + SelT<SEL>::w1 * __popc(c.cm1 & X3) +
             SelT<SEL>::w2 * __popc(c.cm2 & X3);
        t2b = SelT<SEL>::w12 * __popc(X2) - inc + SelT<SEL>::w0 * __popc(c.cm0 & X2) + SelT<SEL>::w1 * __popc(c.cm1 & X2) +
              SelT<SEL>::w2 * __popc(c.cm2 & X2);
        lpb = c.laneC + SelT<SEL>::w12 * __popc(X1) + SelT<SEL>::w0 * __popc(c.cm0 & X1) + SelT<SEL>::w1 * __popc(c.cm1 & X1) +
              SelT<SEL>::w2 * __popc(c.cm2 & X1);
        m31 = (SelT<SEL>::w12 != 0 && (SelT<SEL>::useU || e31)) ? 1 : 0;
        A = st.acc;
        wcol = sh().twp + b;
    } else {
        const uint32_t X3 = st.bm[J3], X2 = st.bm[J2], X1 = st.bm[J1];
        t3 = __popc(c.cm0 & X3) * c.xs + __popc(c.cm12 & X3);
        t2b = __popc(c.cm0 & X2) * c.xs + __popc(c.cm12 & X2);
        lpb = __popc(c.cm0 & X1) * c.xs + __popc(c.cm12 & X1);
        m31 = e31 ? 1 : 0;
        A = st.acc * c.xs + st.acc2;
        wcol = sh().tdl + b;
    }
    int2 *L3 = sh().wl[c.warp].l3 + c.g * W;
    const uint32_t n3 = (uint32_t)__popc(cand3);
    const bool okb = ((c.F & ~st.U & alw<SEL>(st.al[J1])) >> b) & 1u;
    const uint32_t cand2b = c.F & ~st.U & alw<SEL>(st.al[J2]);
    __syncwarp(c.gmask);  // previous readers of the k-3 list and of dense[0] are done
    if ((cand3 >> b) & 1u) L3[__popc(cand3 & ((1u << b) - 1u))] = make_int2((int)b, t3);
    uint32_t colT[W / 2];
    stat_col<W, SEL>(c, stat_entry<W, SEL>(c, (cand2b >> b) & 1u, t2b), colT);  // syncs the group
    const unsigned long long fbase = pack_f<K>(st);
    const bool dep = d32 || d31 || d21;
    if constexpr (SelT<SEL>::cta) bst.thr = max(bst.thr, sh().cthr);
    const uint32_t Mb = d21 ? ((1u << b) - 1u) : ~(1u << b);  // valid v of this lane given f(k-1) = b
    if (!dep && okb) {
        const uint32_t nb = ~(1u << b);
        bst.cnt += (uint32_t)(__popc(cand3 & nb) * __popc(cand2b & nb) - __popc(cand3 & cand2b & nb));
    }
    if constexpr (!SelT<SEL>::lin) {
        // the next v3's list entry and w(v3, b) are loaded one iteration
        // ahead (the LDS -> LDS -> base chain is off the scan's critical path;
        // `& 31` keeps the read in bounds when the list is empty)
        int2 e3n = L3[0];
        int w3n = wcol[((uint32_t)e3n.x & 31u) * 32];
        for (uint32_t i = 0; i < n3; ++i) {
            const int2 e3 = e3n;
            const int w3 = w3n;
            e3n = L3[min(i + 1u, n3 - 1u)];
            w3n = wcol[((uint32_t)e3n.x & 31u) * 32];
            const uint32_t v3 = (uint32_t)e3.x;
            const bool laneok = okb && b != v3 && (!d31 || b > v3);
            const int base = A + e3.y + lpb + m31 * w3;
            const uint32_t row = v3 * (2u * W);  // byte offset of row v3
            if (dep) {
                const uint32_t cand2 = cand2b & ~(1u << v3) & (d32 ? (0xFFFFFFFEu << v3) : kFull);
                bst.cnt += laneok ? (uint32_t)__popc(Mb & cand2) : 0u;
            }
            int raw = scan_row_max<W>(row, colT, base, c.negk);
            if (laneok && raw >= bst.thr) {  // rank >= the lane's best score: filter, then rescan for the v
                const uint32_t cand2 = cand2b & ~(1u << v3) & (d32 ? (0xFFFFFFFEu << v3) : kFull);
                if (!sens_may_win<W>(c, bst, raw, st.U | (1u << v3) | (1u << b), cand2 & Mb)) continue;
                raw = scan_row_tie<W>(row, colT, base, c.one, c.negk);
                const uint32_t bestv = 31u - (uint32_t)(raw & 31);
                const unsigned long long fpack =
                    fbase | ((unsigned long long)v3 << (8 * J3)) | ((unsigned long long)bestv << (8 * J2));
                consider<W, K, false, true>(c, bst, st.U | (1u << v3) | (1u << bestv) | (1u << b), fpack,
                                            (uint32_t)(raw >> 5) - 1u);
            }
        }
        return;
    } else {
        for (uint32_t i = 0; i < n3; i += 2) {
            const bool hasB = i + 1 < n3;
            const int2 eA = L3[i], eB = L3[hasB ? i + 1 : i];
            const int wA = wcol[(uint32_t)eA.x * 32], wB = wcol[(uint32_t)eB.x * 32];
            const uint32_t vA = (uint32_t)eA.x, vB = (uint32_t)eB.x;
            const bool okA = okb && b != vA && (!d31 || b > vA);
            const bool okB = hasB && okb && b != vB && (!d31 || b > vB);
            const int offA = (A + eA.y + lpb + m31 * wA + 1 - c.ishift) * 32;
            const int offB = (A + eB.y + lpb + m31 * wB + 1 - c.ishift) * 32;
            if (dep) {
                const uint32_t cA = cand2b & ~(1u << vA) & (d32 ? (0xFFFFFFFEu << vA) : kFull);
                const uint32_t cB = cand2b & ~(1u << vB) & (d32 ? (0xFFFFFFFEu << vB) : kFull);
                bst.cnt += (uint32_t)(okA ? __popc(Mb & cA) : 0) + (uint32_t)(okB ? __popc(Mb & cB) : 0);
            }
            unsigned iA, iB;
            const unsigned mA = scan_row_thr<W>(vA * (2u * W), colT, bst.thr - offA, iA);
            const unsigned mB = scan_row_thr<W>(vB * (2u * W), colT, bst.thr - offB, iB);
            const bool hitA = okA && mA != iA, hitB = okB && mB != iB;
            if (hitA || hitB) {  // a leaf whose score reaches the lane's / CTA's best score
                if (hitA) {
                    const int best = s16_best(mA) + offA;
                    const uint32_t bestv = 31u - (uint32_t)(best & 31);
                    const unsigned long long fpack =
                        fbase | ((unsigned long long)vA << (8 * J3)) | ((unsigned long long)bestv << (8 * J2));
                    consider<W, K, SelT<SEL>::cta, false>(c, bst, st.U | (1u << vA) | (1u << bestv) | (1u << b), fpack,
                                                          (uint32_t)(best >> 5) - 1u);
                }
                if (hitB) {
                    const int best = s16_best(mB) + offB;
                    if (best >= bst.thr) {
                        const uint32_t bestv = 31u - (uint32_t)(best & 31);
                        const unsigned long long fpack =
                            fbase | ((unsigned long long)vB << (8 * J3)) | ((unsigned long long)bestv << (8 * J2));
                        consider<W, K, SelT<SEL>::cta, false>(c, bst, st.U | (1u << vB) | (1u << bestv) | (1u << b),
                                                              fpack, (uint32_t)(best >> 5) - 1u);
                    }
                }
            }
        }
    }
}

template <int W, int K, int SEL, int J>
__device__ __forceinline__ void level(const Ctx<W> &c, const St<K> &st, Best &bst) {
    if constexpr (K == 1) {
        leaf_k1<W, SEL>(c, bst);
    } else if constexpr (J == K - 2) {
        if constexpr (SelT<SEL>::stat) inners<W, K, SEL>(c, st, c.F & ~st.U & alw<SEL>(st.al[J]), bst);
        else inner<W, K, SEL>(c, st, c.F & ~st.U & alw<SEL>(st.al[J]), bst);
    } else if constexpr (J == K - 3) {
        if constexpr (SelT<SEL>::stat) inner3s<W, K, SEL>(c, st, c.F & ~st.U & alw<SEL>(st.al[J]), bst);
        else inner3<W, K, SEL>(c, st, c.F & ~st.U & alw<SEL>(st.al[J]), bst);
    } else {
        uint32_t cand = c.F & ~st.U & alw<SEL>(st.al[J]);
        while (cand) {
            const uint32_t v = __ffs(cand) - 1;
            cand &= cand - 1u;
            level<W, K, SEL, J + 1>(c, push<W, K, SEL, J>(c, st, v), bst);
        }
    }
}

template <int W, int K>
__device__ __forceinline__ St<K> root(const Ctx<W> &c) {
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
__device__ __forceinline__ bool digits(uint32_t item, int nF, int D, uint32_t (&dg)[kMaxDecode]) {
    uint32_t it = item;
#pragma unroll
    for (int j = kMaxDecode - 1; j >= 0; --j) {
        if (j < D) {
            const uint32_t r = (uint32_t)(nF - j);
            const uint32_t q = __umulhi(it, sh().magic[r]);
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
__device__ __forceinline__ uint32_t descend_range(const Ctx<W> &c, const St<K> &st, const uint32_t (&dg)[kMaxDecode],
                                                  int D, uint32_t maxn, Best &bst) {
    if constexpr (J >= DMAX || J > K - 2) {
        return maxn;  // unreachable: D <= DMAX <= K-1
    } else {
        if (J < D - 1) {
            const uint32_t v = nth_set(c.F & ~st.U, dg[J]);
            if (SelT<SEL>::canon && !((st.al[J] >> v) & 1u)) {
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
            return descend_range<W, K, SEL, J + 1, DMAX>(c, push<W, K, SEL, J>(c, st, v), dg, D, maxn, bst);
        } else {
            uint32_t cand = c.F & ~st.U;
            const uint32_t p = nth_set(cand, dg[J]);
            cand &= ~((1u << p) - 1u);  // raw candidates from the current item on
            uint32_t n = (uint32_t)__popc(cand);
            if (maxn < n) {
                cand &= (1u << nth_set(cand, maxn)) - 1u;
                n = maxn;
            }
            cand &= alw<SEL>(st.al[J]);
            if constexpr (J == K - 2) {
                if constexpr (SelT<SEL>::stat) inners<W, K, SEL>(c, st, cand, bst);
                else inner<W, K, SEL>(c, st, cand, bst);
            } else if constexpr (J == K - 3) {
                if constexpr (SelT<SEL>::stat) inner3s<W, K, SEL>(c, st, cand, bst);
                else inner3<W, K, SEL>(c, st, cand, bst);
            } else {
                while (cand) {
                    const uint32_t v = __ffs(cand) - 1;
                    cand &= cand - 1u;
                    level<W, K, SEL, J + 1>(c, push<W, K, SEL, J>(c, st, v), bst);
                }
            }
            return n;
        }
    }
}

// Items [lo, hi) of depth D (D = 0 only for K = 1).
template <int W, int K, int SEL, int DMAX>
__device__ __forceinline__ void run_range(const Ctx<W> &c, uint32_t lo, uint32_t hi, int D, Best &bst) {
    if constexpr (K == 1) {
        if (lo == 0 && hi > 0) leaf_k1<W, SEL>(c, bst);
    } else {
        uint32_t i = lo;
        while (i < hi) {
            uint32_t dg[kMaxDecode];
            if (!digits(i, c.nF, D, dg)) break;
            i += descend_range<W, K, SEL, 0, DMAX>(c, root<W, K>(c), dg, D, hi - i, bst);
        }
    }
}

// Per-query context.  Must be called by the whole warp (uses shuffles); it
// writes this warp's inc_F table.
template <int W>
__device__ __forceinline__ Ctx<W> make_ctx(const DevTopo &topo, const DevPattern &P, int pid, int xs, uint32_t busy,
                                           int sc, bool pack16, bool lin16 = false) {
    const int lane = threadIdx.x & 31;
    Ctx<W> c;
    const uint32_t nmask = topo.n >= 32 ? kFull : ((1u << topo.n) - 1u);
    c.F = ~busy & nmask;
    c.nF = __popc(c.F);
    c.b = lane & (W - 1);
    c.g = lane / W;
    c.warp = (int)(threadIdx.x >> 5);
    c.gmask = W == 32 ? kFull : (((1u << W) - 1u) << (c.g * W));
    const uint4 mine = sh().cm[c.b];
    c.cm0 = mine.x;
    c.cm1 = mine.y;
    c.cm2 = mine.z;
    c.cm12 = mine.y | mine.z;
    // inc_F(b) = sum_{u in F, u != b} w(u,b)
    const int inFb = (c.F >> c.b) & 1u;
    int incb = 12 * (c.nF - inFb) + 38 * __popc(mine.x & c.F) + 13 * __popc(mine.y & c.F) +
               8 * __popc(mine.z & c.F);
    if (c.b >= topo.n) incb = 0;
    if (lane < W) sh().inc[c.warp][c.b] = incb;
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
    c.pid = pid;
    c.xs = xs;
    c.lut = pid * 3 * xs * xs;
    c.one = sh().one;
    c.negk = c.one * -65536;
    sc &= 3;
    const bool useU = sc == SEL_INSENS;
    const int w12 = sc == SEL_BASE ? 0 : 12;
    c.laneC = useU ? -incb : 0;
    c.acc0 = useU ? TF : 0;
    const int n12 = useU ? (K - 1) : (int)P.dback[K - 1];
    c.leafC = w12 * n12 + c.laneC;
    // inner-scan column of this lane (vertex k-1 on device b, vertex k-2 on v):
    //   LIN  col[v] = T[v][b] + 31 - v, T = 32 w (edge k-2~k-1 scored) or 0, kNeg invalid
    //   SENS col[v] = D[v][b], D = census delta (edge k-2~k-1) or 0, + kSent invalid
    const int sh2 = K >= 2 ? 8 * (K - 2) : 0;
    const bool eK = K >= 2 && ((((uint32_t)(c.fb >> sh2)) >> (K - 1)) & 1u);
    const bool dep = K >= 2 && ((((uint32_t)(c.fs >> sh2)) >> (K - 1)) & 1u);
    const bool sens = sc == SEL_SENS;
    const bool eW = w12 != 0 && (useU || eK);
    const int *T = sens ? (eK ? (dep ? sh().tsed : sh().tse) : (dep ? sh().ts0d : sh().ts0))
                        : (eW ? (dep ? sh().twd : sh().tw) : (dep ? sh().tzd : sh().tz));
#pragma unroll
    for (int v = 0; v < W; ++v) c.col[v] = sens ? T[v * 32 + c.b] : T[v * 32 + c.b] + 31 - v;
    c.colmax = kNeg;
#pragma unroll
    for (int v = 0; v < W; ++v) c.colmax = max(c.colmax, c.col[v]);
    c.ishift = 0;
    c.irange = 0;
    if (lin16) {
        // Eq. 3 table entries t2(v) = sum_U w(u, v) - inc_F(v) are shifted by
        // max_{v in F} inc_F(v) to be >= 0 (the caller's base subtracts it)
        int im = useU && inFb ? incb : 0, imn = useU && inFb ? incb : 0x7FFFFFFF;
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) {
            im = max(im, __shfl_xor_sync(kFull, im, o, W));
            imn = min(imn, __shfl_xor_sync(kFull, imn, o, W));
        }
        c.ishift = im;
        c.irange = useU ? im - min(imn, im) : 0;
#pragma unroll
        for (int j = 0; j < W / 2; ++j) {
            const int lo = c.col[2 * j] < 0 ? kNeg16C : c.col[2 * j];
            const int hi = c.col[2 * j + 1] < 0 ? kNeg16C : c.col[2 * j + 1];
            c.col[j] = (lo & 0xFFFF) | (hi << 16);
        }
    }
    if (pack16) {  // SelT::pack16: col[j] = col(2j) | col(2j+1) << 16 (byte offsets < 2^16)
#pragma unroll
        for (int j = 0; j < W / 2; ++j) c.col[j] = (c.col[2 * j] & 0xFFFF) | (c.col[2 * j + 1] << 16);
    }
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

// Shared tables for Eq. 2 row stride xs + npats Eq. 2 tables + edge lists.
// Caller syncs.
// Pair tables a single-query kernel reads (indices into the ten of Shared,
// order tw tz twd tzd twp tdl tse tsed ts0 ts0d): the lane column's table
// (make_ctx) and the k-3 weight / census-delta table (inner3).
__device__ __forceinline__ int col_table(int sc, const DevPattern &P) {
    const int K = P.k, base = sc & 3;
    const int sh2 = K >= 2 ? 8 * (K - 2) : 0;
    const bool eK = K >= 2 && ((P.fwd_back[K - 2] >> (K - 1)) & 1u);
    const bool dep = K >= 2 && (((*reinterpret_cast<const uint64_t *>(P.fwd_src) >> sh2) >> (K - 1)) & 1u);
    if (base == SEL_SENS) return eK ? (dep ? 7 : 6) : (dep ? 9 : 8);
    const bool eW = base != SEL_BASE && (base == SEL_INSENS || eK);
    return eW ? (dep ? 2 : 0) : (dep ? 3 : 1);
}

template <int MAXP, int LUTCAP>
__device__ __forceinline__ void load_shared(const Tables<MAXP, LUTCAP> &tb, int xs, int ub_r2 = -1, int only_sc = -1,
                                            int *lut = nullptr, int regions = 3) {
    Shared &s = sh();
    const DevTopo &topo = tb.topo;
    const int tid = threadIdx.x;
    if (tid < kMaxN) s.cm[tid] = make_uint4(topo.cm[tid][0], topo.cm[tid][1], topo.cm[tid][2], topo.cm[tid][3]);
    if (tid == 0) {
        s.one = 1;
        s.cthr = 32;
        s.ckey = 0ull;
    }
    if (tid <= kMaxN) s.magic[tid] = tid >= 2 ? (0xFFFFFFFFu / (uint32_t)tid + 1u) : 0u;
    static_assert(offsetof(Shared, ts0d) == offsetof(Shared, tw) + 9 * kNN * sizeof(int), "pair tables contiguous");
    if (tb.pre && only_sc >= 0) {
        // single query: only the two tables this selector / pattern reads (8 KB
        // of the 40-KB image; the prologue is the fixed cost of every launch)
        const int t0 = col_table(only_sc, tb.pat[0]), t1 = (only_sc & 3) == SEL_SENS ? 5 : 4;
        int4 *dst = reinterpret_cast<int4 *>(s.tw);
        for (int i = tid; i < 2 * kNN / 4; i += blockDim.x) {
            const int t = i < kNN / 4 ? t0 : t1, j = i & (kNN / 4 - 1);
            dst[t * (kNN / 4) + j] = tb.pre[t * (kNN / 4) + j];
        }
    } else if (tb.pre) {
        // cached image (host-built once per topology and xs): 16-B loads from L2
        int4 *dst = reinterpret_cast<int4 *>(s.tw);
        for (int i = tid; i < kPairTables * kNN / 4; i += blockDim.x) dst[i] = tb.pre[i];
    } else {
        int *pt = &s.tw[0];  // the ten tables, contiguous (asserted above)
        for (int i = tid; i < kNN; i += blockDim.x) {
            int e[kPairTables];
            pair_table_entry(topo, i, xs, e);
#pragma unroll
            for (int t = 0; t < kPairTables; ++t) pt[t * kNN + i] = e[t];
        }
    }
    if (!lut) lut = sh_lut();  // single-query Eq. 2 kernels pass lut1()
    // single-query additive kernels read no Eq. 2 table (and get no dynamic
    // shared memory for it: smem_single)
    const int nlut = only_sc >= 0 && (only_sc & 3) != SEL_SENS ? 0 : tb.npats;
    for (int p = 0; p < tb.npats; ++p) {
        const DevPattern &P = tb.pat[p];
        const uint16_t *rank = tb.lut + P.lut_off;
        const int m = P.m;
        for (int i = tid; p < nlut && i < regions * xs * xs; i += blockDim.x) {
            const int x = i / xs, y = i % xs;
            int v = kNeg;
            if (i < xs * xs) v = (x + y <= m) ? ((int)rank[x * (m + 1) + y] + 1) * 32 : 0;
            lut[p * regions * xs * xs + i] = v;
        }
        if (tid < 28) s.edge[p][tid] = P.edge[tid];
    }
    if (ub_r2 >= 0) {
        // prune mode, Eq. 2 (single pattern): ubtab[x*xs + y] = max rank entry
        // over the censuses reachable from (x, y) by ub_r2 more edges
        __syncthreads();
        const int m = tb.pat[0].m;
        int *ub = lut + 3 * xs * xs;
        for (int i = tid; i < xs * xs; i += blockDim.x) {
            const int x = i / xs, y = i % xs;
            int best = 0;
            for (int dx = 0; dx <= ub_r2; ++dx)
                for (int dy = 0; dx + dy <= ub_r2; ++dy)
                    if (x + dx + y + dy <= m && x + dx < xs && y + dy < xs) best = max(best, lut[(x + dx) * xs + y + dy]);
            ub[i] = best;
        }
    }
}

// Static tables of the SelT::stat kernels (StatShared), from the pair tables
// load_shared put in shared memory (the lane column's table and twp / tdl).
// Caller syncs before (tables loaded) and after.
template <int W, int SEL>
__device__ __forceinline__ void build_stat(const DevPattern &P, int xs) {
    const int K = P.k, tid = threadIdx.x;
    const bool e32 = K >= 3 && ((P.fwd_back[K - 3] >> (K - 2)) & 1u);
    const bool d32 = SelT<SEL>::canon && K >= 3 && ((P.fwd_src[K - 3] >> (K - 2)) & 1u);
    const int *ct = &sh().tw[0] + col_table(SEL & 3, P) * kNN;
    const int *dt = SelT<SEL>::lin ? sh().twp : sh().tdl;
    const bool m32 = SelT<SEL>::lin ? (SelT<SEL>::w12 != 0 && (SelT<SEL>::useU || e32)) : e32;
    constexpr int H = W / 2;
    for (int i = tid; i < (W + 1) * H; i += blockDim.x) {
        const int v3 = i / H, q = i % H;
        uint32_t pr = 0;
        if (v3 < W) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int v = 2 * q + h;
                const bool bad = v == v3 || (d32 && v <= v3);
                int e;
                if constexpr (SelT<SEL>::lin16) e = bad ? kStY : (m32 ? 32 * dt[v3 * 32 + v] : 0);
                else e = 4 * ((m32 ? dt[v3 * 32 + v] : 0) + (bad ? xs * xs : 0));
                pr |= ((uint32_t)e & 0xFFFFu) << (16 * h);
            }
        }
        stt<SelT<SEL>::pack16>().row[i] = pr;
    }
    for (int i = tid; i < H * W; i += blockDim.x) {
        const int q = i / W, b = i % W;
        uint32_t pr = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int v = 2 * q + h;
            const int t = ct[v * 32 + b];
            int e;
            if constexpr (SelT<SEL>::lin16) e = t == kNegTable ? kStZ : t + 31 - v;
            else e = t;
            pr |= ((uint32_t)e & 0xFFFFu) << (16 * h);
        }
        stt<SelT<SEL>::pack16>().col[i] = pr;
    }
}

// CTAs per SM the single-query kernels are compiled for: three for the static
// lin16 Greedy kernels (80 registers, a few spills outside the hot loop; C4
// 84.8 -> 82.9 us), two otherwise (the Eq. 3 kernel spilled more at 80
// registers and ran 3 % slower)
template <int SEL>
constexpr int kCtasPerSm = SelT<SEL>::stat && SelT<SEL>::lin16 && SelT<SEL>::base == SEL_GREEDY ? 3 : 2;

// ---------------------------------------------------------------- single query
// Items = prefixes of depth D, in chunks of `chunk` consecutive items; local
// chunk q of rank r is global chunk q*world + r.  Group g of a warp walks the
// g-th slice of the chunk.
template <int W, int K, int SEL>
__global__ void __launch_bounds__(kBlock, kCtasPerSm<SEL>)
esa_single(const __grid_constant__ SingleTables tb, const mapa_query *__restrict__ dq,
           mapa_record *__restrict__ rec, int D, int rank, int world, int stripe) {
    constexpr int G = 32 / W;
    constexpr int DMAX = (K - 1) < kMaxDecode ? (K - 1) : kMaxDecode;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int xs = tb.xs;
    int ub_r2 = -1;
    if constexpr (SelT<SEL>::prune && SelT<SEL>::base == SEL_SENS && K >= 4) {
        // edges a k-2 scan adds: k-2's back edges + the edge (k-2, k-1)
        const DevPattern &P = tb.pat[0];
        ub_r2 = (int)P.dback[K - 2] + (int)((P.fwd_back[K - 2] >> (K - 1)) & 1u);
    }
    // the query load is issued first: its latency overlaps the table copy
    const uint32_t busy = *reinterpret_cast<const volatile uint32_t *>(&dq->busy);
    if constexpr (SelT<SEL>::pack16 || SelT<SEL>::stat) {
        // the static tables must sit where the immediates point (see kLut1Addr)
        if ((uint32_t)__cvta_generic_to_shared(stat_base<SelT<SEL>::pack16>()) != kLut1Addr) {
            if (tid == 0) atomicExch(&rec->status, 2u);
            return;
        }
    }
    if constexpr (SelT<SEL>::pack16) {
        // (static path: an index carries up to three sentinels -> 4 regions)
        load_shared(tb, xs, ub_r2, SEL & 3, lut1(), SelT<SEL>::stat ? 4 : 3);
    } else {
        load_shared(tb, xs, ub_r2, SEL & 3);
    }
    __syncthreads();
    if constexpr (SelT<SEL>::stat) {
        build_stat<W, SEL>(tb.pat[0], xs);
        __syncthreads();
    }

    Ctx<W> c = make_ctx<W>(tb.topo, tb.pat[0], 0, xs, busy, SEL & 3, SelT<SEL>::pack16, SelT<SEL>::lin16);
    if constexpr (SelT<SEL>::lin16) {
        // the host chose 16-bit scans from busy_hint; a query whose free set
        // breaks the range (lin16_fits) is refused loudly, never mis-scored
        if (32 * (50 * (K - 2) + c.irange) > (SelT<SEL>::stat ? kStTmax : kLin16Max)) {
            if (tid == 0) atomicExch(&rec->status, 1u);
            return;
        }
    }

    // Rank r owns the stripes s = r, r + world, ... of `stripe` consecutive
    // items; its local item space is their concatenation.  Warps grab local
    // chunks by guided self-scheduling (size = remaining / (2 x warps), at
    // least 2G), so few chunks are decoded and the tail stays short.
    const uint32_t N = (K <= c.nF) ? perm_count(c.nF, D) : 0u;
    const uint32_t L = (uint32_t)stripe;
    const uint32_t nS = (N + L - 1u) / L;
    const uint32_t myS = nS > (uint32_t)rank ? (nS - (uint32_t)rank + (uint32_t)world - 1u) / (uint32_t)world : 0u;
    const bool ownLast = nS > 0 && ((nS - 1u) % (uint32_t)world) == (uint32_t)rank;
    const uint32_t Nloc = myS == 0 ? 0u : (ownLast ? (myS - 1u) * L + (N - (nS - 1u) * L) : myS * L);
    const uint32_t P = gridDim.x * (uint32_t)kWarps;
    Best bst{0ull, 0u, 0u, 32, 0u, 32, SelT<SEL>::prune ? reinterpret_cast<unsigned *>(&rec->reserved) : nullptr};
    const uint32_t g = (uint32_t)(lane / W);
    // The first chunk of every warp is static (warp w takes [w s0, (w+1) s0)),
    // so a launch starts without P same-address atomics; the counter then
    // hands out [off0, Nloc), and a warp that reads it exhausted leaves
    // without an atomic.
    // (chunks of at least one item per group and two per warp: a minimum of
    // two items per GROUP left warps of the W <= 16 kernels idle on queries
    // with few prefixes -- cubemesh16 k = 8 at 12 free: 62 -> 51 us; W = 32
    // keeps two per warp, measured no better with one)
    const uint32_t cmin = max(2u, (uint32_t)G);
    const uint32_t s0 = (max(cmin, Nloc / (2u * P)) + G - 1u) / G * G;
    const uint32_t off0 = (uint32_t)min((unsigned long long)P * s0, (unsigned long long)Nloc);
    const uint32_t gw = blockIdx.x * (uint32_t)kWarps + (uint32_t)warp;
    bool first = true;
    for (;;) {
        uint32_t start = Nloc, sz = 0;
        if (first) {
            first = false;
            if (gw * s0 >= off0) continue;  // no static chunk: straight to the counter
            start = gw * s0;
            sz = s0;
        } else {
            if (off0 >= Nloc) break;  // the static chunks covered every item: no counter round trip
            if (lane == 0) {
                const uint32_t cur = off0 + ld_relaxed(&rec->ctr);
                if (cur < Nloc) {
                    sz = max(cmin, (Nloc - cur) / (2u * P));
                    sz = (sz + G - 1u) / G * G;
                    start = off0 + atomicAdd(&rec->ctr, sz);
                }
            }
            start = __shfl_sync(kFull, start, 0);
            sz = __shfl_sync(kFull, sz, 0);
        }
        if (start >= Nloc) break;
        const uint32_t end = min(start + sz, Nloc);
        const uint32_t per = (end - start + G - 1u) / G;
        uint32_t j0 = start + g * per;
        const uint32_t j1 = min(j0 + per, end);
        while (j0 < j1) {  // split at stripe boundaries
            const uint32_t sl = j0 / L;
            const uint32_t seg = min(j1, (sl + 1u) * L);
            const uint32_t lo = (sl * (uint32_t)world + (uint32_t)rank) * L + (j0 - sl * L);
            run_range<W, K, SEL, DMAX>(c, lo, lo + (seg - j0), D, bst);
            j0 = seg;
        }
        __syncwarp();
    }
    unsigned long long key = bst.key, cnt = bst.cnt;
    warp_reduce(key, cnt);
    if (lane == 0) {
        sh().key[warp] = key;
        sh().cnt[warp] = cnt;
    }
    __syncthreads();
    if (warp == 0) {
        key = lane < kWarps ? sh().key[lane] : 0ull;
        cnt = lane < kWarps ? sh().cnt[lane] : 0ull;
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
__device__ __forceinline__ void batch_item(const Ctx<W> &c, uint32_t j, Best &bst) {
    if constexpr (SelT<SEL>::lin16 && K < 3) {
        return;  // never dispatched (lin16 from k = 3)
    } else if constexpr (K == 1) {
        if (j == 0) leaf_k1<W, SEL>(c, bst);
    } else {
        if (j < (uint32_t)c.nF) run_range<W, K, SEL, 1>(c, j, j + 1, 1, bst);
    }
}

template <int W, int SEL>
__device__ __forceinline__ void batch_dispatch_k(int K, const Ctx<W> &c, uint32_t j, Best &bst) {
    switch (K) {
        case 1: batch_item<W, 1, SEL>(c, j, bst); break;
        case 2: batch_item<W, 2, SEL>(c, j, bst); break;
        case 3: batch_item<W, 3, SEL>(c, j, bst); break;
        case 4: batch_item<W, 4, SEL>(c, j, bst); break;
        case 5: batch_item<W, 5, SEL>(c, j, bst); break;
        case 6: batch_item<W, 6, SEL>(c, j, bst); break;
        case 7: batch_item<W, 7, SEL>(c, j, bst); break;
        case 8: batch_item<W, 8, SEL>(c, j, bst); break;
        default: break;
    }
}

__device__ __forceinline__ bool key_fits(int W, const DevPattern &P) { return 15 + W + P.eb <= 63; }

template <int W, int CANON>
__global__ void __launch_bounds__(kBlock, 2)
esa_batch(const __grid_constant__ MultiTables tb, long long nq, const mapa_query *__restrict__ qs,
          mapa_record *__restrict__ res, uint32_t *__restrict__ ctr, const uint32_t *__restrict__ perm) {
    constexpr int G = 32 / W;
    const int lane = threadIdx.x & 31;
    const int xs = tb.xs;
    load_shared(tb, xs);
    __syncthreads();

    const unsigned long long nslots = (unsigned long long)nq * W;
    const uint32_t g = (uint32_t)(lane / W);
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(reinterpret_cast<unsigned long long *>(ctr), (unsigned long long)G);
        base = __shfl_sync(kFull, base, 0);
        if (base >= nslots) break;
        // G | W: every group of the warp has the same query.  Queries are taken
        // in `perm` order (bucketed by code path: consecutive warps run the same
        // (K, selector) instantiation, which keeps the instruction cache warm)
        const unsigned long long q = perm ? (unsigned long long)perm[base / W] : base / W;
        const mapa_query qu = qs[q];
        const uint32_t pid = qu.pattern;
        if (pid >= (uint32_t)tb.npats || !key_fits(W, tb.pat[pid < (uint32_t)tb.npats ? pid : 0])) {
            if (lane == 0 && (base % W) == 0) atomicExch(&res[q].status, 1u);
            continue;
        }
        const DevPattern &P = tb.pat[pid];
        const int scq = sel_code(qu.selector, qu.sensitive);
        // 16-bit scans (two leaves per VIADDMNMX.S16x2) for the additive
        // selectors when this query's free set keeps every sum in range (the
        // single-query kernels' lin16, decided here per query, exactly)
        bool l16 = W >= 16 && P.k >= 3 && (scq == SEL_GREEDY || scq == SEL_INSENS);
        Ctx<W> c = make_ctx<W>(tb.topo, P, (int)pid, xs, qu.busy, scq, false, l16);
        if (l16 && 32 * (50 * (P.k - 2) + c.irange) > kLin16Max) {
            l16 = false;
            c = make_ctx<W>(tb.topo, P, (int)pid, xs, qu.busy, scq, false, false);
        }
        if (P.k > c.nF) continue;
        const uint32_t j = (uint32_t)(base % W) + g;
        Best bst{0ull, 0u, 0u, 32, 0u, 32, nullptr};
        switch (scq) {
            case SEL_GREEDY:
                if (W >= 16 && l16) batch_dispatch_k<W, SEL_GREEDY | 4 * CANON | 8 | 32 * (W >= 16)>(P.k, c, j, bst);
                else batch_dispatch_k<W, SEL_GREEDY | 4 * CANON | 8>(P.k, c, j, bst);
                break;
            case SEL_INSENS:
                if (W >= 16 && l16) batch_dispatch_k<W, SEL_INSENS | 4 * CANON | 8 | 32 * (W >= 16)>(P.k, c, j, bst);
                else batch_dispatch_k<W, SEL_INSENS | 4 * CANON | 8>(P.k, c, j, bst);
                break;
            case SEL_SENS: batch_dispatch_k<W, SEL_SENS | 4 * CANON | 8>(P.k, c, j, bst); break;
            default: batch_dispatch_k<W, SEL_BASE | 4 * CANON | 8>(P.k, c, j, bst); break;
        }
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
__device__ __forceinline__ void trace_items(const Ctx<W> &c, int D, uint32_t nItems, uint32_t gid, uint32_t ngroups,
                                            Best &bst) {
    constexpr int DMAX = (K - 1) < 2 ? (K - 1) : 2;
    const uint32_t per = (nItems + ngroups - 1u) / ngroups;
    const uint32_t lo = gid * per, hi = min(lo + per, nItems);
    if (lo < hi) run_range<W, K, SEL, DMAX>(c, lo, hi, D, bst);
}

template <int W, int SEL>
__device__ __forceinline__ void trace_dispatch_k(int K, const Ctx<W> &c, int D, uint32_t nItems, uint32_t gid,
                                                 uint32_t ngroups, Best &bst) {
    switch (K) {
        case 1: trace_items<W, 1, SEL>(c, D, nItems, gid, ngroups, bst); break;
        case 2: trace_items<W, 2, SEL>(c, D, nItems, gid, ngroups, bst); break;
        case 3: trace_items<W, 3, SEL>(c, D, nItems, gid, ngroups, bst); break;
        case 4: trace_items<W, 4, SEL>(c, D, nItems, gid, ngroups, bst); break;
        case 5: trace_items<W, 5, SEL>(c, D, nItems, gid, ngroups, bst); break;
        case 6: trace_items<W, 6, SEL>(c, D, nItems, gid, ngroups, bst); break;
        case 7: trace_items<W, 7, SEL>(c, D, nItems, gid, ngroups, bst); break;
        case 8: trace_items<W, 8, SEL>(c, D, nItems, gid, ngroups, bst); break;
        default: break;
    }
}

// One CTA per trace; ALLOC / RELEASE ops in order; the busy mask lives in
// shared memory (§3.6 state management), decisions go to HBM as keys.
template <int W, int CANON>
__global__ void __launch_bounds__(kBlock, 1)
esa_trace(const __grid_constant__ MultiTables tb, int nops, const mapa_trace_op *__restrict__ ops, int njobs,
          const mapa_query *__restrict__ jobs, unsigned long long *__restrict__ keys) {
    constexpr int G = 32 / W;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x;
    const int xs = tb.xs;
    load_shared(tb, xs);
    if (tid == 0) sh().busy = 0u;
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
        const int ep = okp ? (int)pid : 0;
        const DevPattern &P = tb.pat[ep];
        if (cur.op == 0) {
            const uint32_t busy = sh().busy;
            // Topo-aware (SPEC select_topo_aware; reading A21): the device set
            // is the k lowest free ids of the smallest partition (recursive
            // socket bisection, host table) with >= k free devices, else the k
            // lowest free ids overall; its mapping is Baseline's (lex-smallest
            // edge list), found by enumerating that set alone.
            const bool topo = qu.selector == MAPA_SEL_TOPO;
            uint32_t ebusy = busy;
            if (topo) {
                if (tid == 0) {
                    const uint32_t nm = tb.topo.n >= 32 ? kFull : ((1u << tb.topo.n) - 1u);
                    const uint32_t Fr = ~busy & nm;
                    uint32_t from = Fr;
                    for (int q = 0; q < tb.npart; ++q)
                        if (__popc(tb.part[q] & Fr) >= (int)P.k) { from = tb.part[q] & Fr; break; }
                    uint32_t S = 0;
                    for (int q = 0; q < (int)P.k && from; ++q) { S |= from & (0u - from); from &= from - 1u; }
                    sh().topoS = (__popc(S) == (int)P.k) ? S : 0u;
                }
                __syncthreads();
                ebusy = ~sh().topoS;
            }
            const int scode = topo ? SEL_BASE : sel_code(qu.selector, qu.sensitive);
            Ctx<W> c = make_ctx<W>(tb.topo, P, ep, xs, ebusy, scode, false);
            Best bst{0ull, 0u, 0u, 32, 0u, 32, nullptr};
            if (okp && P.k <= c.nF) {
                const int D = (P.k - 1) < 2 ? (P.k - 1) : 2;
                const uint32_t nItems = perm_count(c.nF, D);
                switch (scode) {
                    case SEL_GREEDY: trace_dispatch_k<W, SEL_GREEDY | 4 * CANON | 8>(P.k, c, D, nItems, gid, kWarps * G, bst); break;
                    case SEL_INSENS: trace_dispatch_k<W, SEL_INSENS | 4 * CANON | 8>(P.k, c, D, nItems, gid, kWarps * G, bst); break;
                    case SEL_SENS: trace_dispatch_k<W, SEL_SENS | 4 * CANON | 8>(P.k, c, D, nItems, gid, kWarps * G, bst); break;
                    default: trace_dispatch_k<W, SEL_BASE | 4 * CANON | 8>(P.k, c, D, nItems, gid, kWarps * G, bst); break;
                }
            }
            __syncwarp();
            unsigned long long key = bst.key, cnt = bst.cnt;
            warp_reduce(key, cnt);
            if (lane == 0) sh().key[warp] = key;
            __syncthreads();
            if (tid == 0) {
                unsigned long long best = 0;
                for (int w = 0; w < kWarps; ++w) best = sh().key[w] > best ? sh().key[w] : best;
                ky[cur.job] = best;
                if (best) sh().busy = busy | (__brev((uint32_t)(best >> P.eb) & wmask) >> (32 - W));
            }
        } else {
            if (tid == 0) {
                const unsigned long long kk = ky[cur.job];
                sh().busy &= ~(__brev((uint32_t)(kk >> P.eb) & wmask) >> (32 - W));
            }
        }
        __syncthreads();
    }
}

template <int MAXP, int LUTCAP>
int smem_bytes(const Tables<MAXP, LUTCAP> &tb) {
    return (int)sizeof(Shared) + (tb.npats * 3 + 1) * tb.xs * tb.xs * (int)sizeof(int);
}

// dynamic shared memory of a single-query kernel: the additive selectors read
// no Eq. 2 table, the Eq. 2 kernels keep theirs in static memory (g_stL)
inline int smem_single(int sc, int smem) { return (sc & 3) == SEL_SENS ? smem : (int)sizeof(Shared); }

inline int set_smem(const void *f, int bytes) {
    return (int)cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace
}  // namespace mapa
