// internal.h — structs shared by the host side (mapa_host.cpp) and the
// sm_100a kernels (esa.cu) of libmapa.  Not part of the C-ABI.
#pragma once

#include <cstdint>
#include <string>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

#include "../../include/mapa.h"

namespace mapa {

constexpr int kMaxK = 8;        // narrow path (packed 63-bit key)
constexpr int kMaxKDeep = 16;   // deep path (256-bit key)
constexpr int kMaxEdges = 120;  // C(16,2)
constexpr int kMaxTup = 2048;   // deep path: suffix index tuples per launch
constexpr int kMaxN = 32;        // narrow path (u32 masks)
constexpr int kMaxNDeep = 64;   // deep path (u64 masks)
constexpr int kMaxPats = 16;      // patterns per batch / trace launch
constexpr int kLutCapSingle = 1024;  // (m+1)^2 <= 841 for m <= 28
constexpr int kLutCapMulti = 4096;

// Link class codes (Table 1): 0 = DoubleNVLink2 50, 1 = SingleNVLink2 25,
// 2 = SingleNVLink1 20, 3 = PCIe 12 (also the fallback for unlinked pairs).
constexpr int kClassBw[4] = {50, 25, 20, 12};

// Device view of a topology: per device v the class masks
//   cm[v].x = {u : class(u,v) == 0}, .y = class 1, .z = class 2, .w = class 3
// (u != v, u < n).  The masks of a device partition the other devices, so
//   sum_{u in X} w(u,v) = 12|X| + 38 popc(x&X) + 13 popc(y&X) + 8 popc(z&X)
// for any X not containing v (weights 50,25,20,12 = 12 + {38,13,8,0}).
struct DevTopo {
    uint32_t cm[kMaxN][4];
    int32_t n;
    int32_t width;  // 8, 16 or 32 lanes per group
};

// Device view of a compiled pattern.  Vertex order = pattern index order
// (the order of the mapping tuple whose lex-min the canonical mode keeps).
// The three byte arrays are read as one 64-bit word each: keep them 8-aligned.
struct alignas(8) DevPattern {
    uint8_t fwd_back[8];        // fwd_back[j] bit u (u > j): pattern edge (j,u)
    uint8_t fwd_src[8];         // fwd_src[j] bit u (u > j): lex-leader f(j) < f(u)
    uint8_t dback[8];           // |{i < j : (i,j) in E}|
    uint8_t k, m, clique, eb;   // eb = C(k,2)
    uint16_t lut_off;           // offset of the Eq. 2 rank table in the LUT pool
    uint16_t aut;               // |Aut(P)|
    uint8_t edge[28];           // a | b << 4, a < b
    uint8_t pad[4];
};
static_assert(sizeof(DevPattern) == 64, "DevPattern layout");

// The ten 32x32 pair tables of the narrow kernels' shared memory (order and
// meaning: esa_kernels.cuh `Shared`), built per CTA, or copied from a cached
// device image built once per (topology, Eq. 2 row stride) on the host.
constexpr int kNegTable = -(1 << 28);

#ifdef __CUDACC__
// Relaxed GPU-scope reads of words other CTAs update with atomics (work
// counters, published bounds).  A `volatile` read compiles to a system-scope
// strong load (LDG.E.STRONG.SYS), which is slower and serialises under
// contention; these are only hints or are re-checked by the atomic that follows.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
#endif
// lin16 single-query scans (16-bit Eq. 1 / Eq. 3): the largest 32 (50 (k-2) +
// inc_F spread) the kernels accept -- the per-v3-table path (prune mode) and
// the static-table path (esa_kernels.cuh, kStX / kStY / kStZ)
constexpr int kLin16Max = 31135;
constexpr int kLin16StatMax = 14768 - 1632;
constexpr int kPairTables = 10;
inline __host__ __device__ void pair_table_entry(const DevTopo &topo, int i, int xs, int out[kPairTables]) {
    const int v = i >> 5, b = i & 31;
    const int sent = xs * xs;
    int w = kNegTable, d = 0;
    if (v != b && v < topo.n && b < topo.n) {
        if ((topo.cm[b][0] >> v) & 1u) { w = 50; d = xs; }
        else if ((topo.cm[b][1] >> v) & 1u) { w = 25; d = 1; }
        else if ((topo.cm[b][2] >> v) & 1u) { w = 20; d = 1; }
        else w = 12;
    }
    const bool bad = w == kNegTable, badd = bad || v >= b;
    out[0] = bad ? kNegTable : 32 * w;            // tw
    out[1] = bad ? kNegTable : 0;                 // tz
    out[2] = badd ? kNegTable : 32 * w;           // twd
    out[3] = badd ? kNegTable : 0;                // tzd
    out[4] = bad ? 0 : w;                         // twp
    out[5] = d;                                   // tdl
    out[6] = 4 * (d + (bad ? sent : 0));          // tse (byte offsets, see scan_dense)
    out[7] = 4 * (d + (badd ? sent : 0));         // tsed
    out[8] = 4 * (bad ? sent : 0);                // ts0
    out[9] = 4 * (badd ? sent : 0);               // ts0d
}

constexpr int kMaxParts = 64;
template <int MAXP, int LUTCAP>
struct Tables {
    DevTopo topo;
    int32_t npats;
    int32_t xs;      // row stride of the Eq. 2 tables on the device (16 if every m <= 15, else 32)
    int32_t npart;   // Topo-aware partitions (trace kernel; SPEC select_topo_aware)
    int32_t pad;
    const int4 *pre; // device image of the ten pair tables for (topo, xs), or null (built per CTA)
    uint32_t part[kMaxParts];  // device masks, smallest first, ties by lowest device
    DevPattern pat[MAXP];
    uint16_t lut[LUTCAP];
};
using SingleTables = Tables<1, kLutCapSingle>;
using MultiTables = Tables<kMaxPats, kLutCapMulti>;

// Kernel selector codes: Greedy (Eq. 1), Preserve-insensitive (Eq. 3),
// Preserve-sensitive (Eq. 2 rank), Baseline (constant score).
enum { SEL_GREEDY = 0, SEL_INSENS = 1, SEL_SENS = 2, SEL_BASE = 3 };
inline __host__ __device__ int sel_code(int selector, int sensitive) {
    return selector == MAPA_SEL_BASELINE ? SEL_BASE
         : selector == MAPA_SEL_PRESERVE ? (sensitive ? SEL_SENS : SEL_INSENS) : SEL_GREEDY;
}

// Canonical-mode patterns get fwd_src from the lex-leader constraints; RAW
// mode zeroes fwd_src (no symmetry breaking).
struct LaunchCfg {
    int grid;
    int block;
    int depth;      // decoded prefix depth D
    int chunk;      // items per counter grab
};

// Deep path (k <= 16): a warp-uniform DFS places vertices 0..T-1 (T = k - L),
// then the lanes scan a table of L-tuples of indices into the r remaining free
// devices (sorted), one tuple per lane.  Tuple word: byte l = i_l.  The
// score of a tuple is A + the sum of NT "terms", each one read of the warp's
// per-node table: a partial pt[l][i_l] (suffix vertex T+l against the placed
// prefix) or a pair value wt[i_a][i_b] (a scored suffix-internal pair).
constexpr int kDeepMaxTerms = 6;
// Eq. 2 deep branch and bound: (k + 1) bound tables of (m + 1)^2 u16 are built
// when they fit in this many entries (34 KB of shared memory)
constexpr int kSensBoundMax = 17408;

struct DeepTables {
    uint64_t cm[kMaxNDeep][3];  // cm[v][c] = {u != v : class(u, v) == c}, c = 0 (50), 1 (25), 2 (20)
    int32_t n;
    int32_t k, m, L, T, r;   // r = free devices left for the suffix at every node
    int32_t ntup;            // valid tuples (suffix-internal lex-leader constraints applied)
    int32_t xsd;             // census index stride m+1 (Eq. 2 table [x*(m+1) + y])
    int32_t clique;
    int32_t nes;             // suffix-internal scored pairs (the pair table is built iff > 0)
    int32_t pcon;            // canonical: per-vertex prefix lower bounds beyond pcommon exist
    int32_t eb;              // C(k,2)
    int32_t pcommon;         // canonical: prefix vertices that are lex-leader sources of EVERY suffix vertex
    int32_t scale;           // the scan compares scale * score (Eq. 3 pair folding: L-1, else 1)
    int32_t nterm;           // terms per tuple (<= kDeepMaxTerms)
    // lanes2 (L = 2 for any r <= 64, no tuple table): vertex T walks the r
    // remaining devices i, vertex T+1 sits on the lanes j (two rounds when r > 32)
    int32_t lanes2;
    int32_t l2e;             // lanes2: the pair (T, T+1) is scored (Eq. 1 / 2 pattern edge, Eq. 3 always)
    int32_t l2dep;           // lanes2, canonical: lex-leader f(T) < f(T+1)
    uint8_t term[kDeepMaxTerms][3];  // (kind 0: pt of suffix vertex a | kind 1: pair (a, b))
    uint8_t pad0[2];
    int32_t tcount[kMaxNDeep + 1];  // tcount[r']: tuples whose indices are all < r' (table sorted by max index)
    uint16_t back[kMaxKDeep];  // back[u] bit j: pattern edge (j, u), j < u
    uint16_t src[kMaxKDeep];   // src[u] bit j: canonical f(j) < f(u) (0 in RAW mode)
    uint8_t edge[kMaxEdges];   // pattern edges a | b << 4
    uint16_t adj[kMaxKDeep];   // pattern adjacency (branch and bound)
    uint8_t c2[kMaxKDeep + 1]; // c2[d]: pattern edges with both endpoints >= d (branch and bound)
    uint8_t pad1[3];
    uint32_t tup[kMaxTup];
};

// Kernel launchers (esa.cu).  Return cudaError_t as int.
// sc = sel_code(...) | 4 * canonical; canon = 1 unless MAPA_F_RAW.
int launch_single(const SingleTables &tb, int sc, const mapa_query *d_query, mapa_record *d_record, int depth,
                  int rank, int world, int stripe, int grid, void *stream);
int launch_batch(const MultiTables &tb, int canon, int64_t nq, const mapa_query *d_queries,
                 mapa_record *d_results, uint32_t *d_ctr, const uint32_t *d_perm, int grid, void *stream);
// Batch query order by code path (counting sort by (k, selector) bucket).
struct BucketKeys {
    int32_t npats;
    uint8_t k[kMaxPats];
};
int launch_bucket(const BucketKeys &bk, int64_t nq, const mapa_query *d_queries, unsigned int *d_cnt,
                  unsigned int *d_cursor, uint32_t *d_perm, void *stream);
int launch_trace(const MultiTables &tb, int canon, int ntraces, int nops, const mapa_trace_op *d_ops, int njobs,
                 const mapa_query *d_jobs, uint64_t *d_keys, void *stream);
// deep path (esa_deep.cu); sc = sel_code | 4 * canonical
int launch_deep(const DeepTables &tb, int sc, const uint16_t *d_lut, const mapa_query64 *d_query,
                mapa_wide_record *d_record, int depth, int rank, int world, int stripe, int grid, void *stream);
int max_blocks_per_sm_deep(int n, int nterm, int sc, int lut_bytes);
int device_sm_count();
int max_blocks_per_sm_single(int width, int k, int sc, int xs);
int max_blocks_per_sm_batch(int width, int canon, int npats, int xs);
const char *cuda_error_string(int err);

}  // namespace mapa
