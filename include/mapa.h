/*
 * mapa.h — C-ABI of libmapa.so, the B200-native MAPA hot path
 * (Multi-Accelerator Pattern Allocation, SC'21, arXiv 2110.03214).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n
 * (section / equation / algorithm named beside each).  Device ids are 0-based
 * here (the paper's and SPEC's 1-based id minus 1; lexicographic order is
 * unchanged).  No C++ exception ever crosses this ABI; every entry point
 * returns a mapa_status and leaves outputs and state untouched on error
 * (S:74).  The message of the last error on the calling thread is available
 * from mapa_last_error().
 *
 * What the hot path computes:
 *   enumerate every injective map f: V(P) -> F of the pattern P into the free
 *   devices F of the hardware graph G (complete; subgraph matching
 *   §3.3), score it (Eq. 1 AggBW P:575-577, Eq. 2 predicted EffBW
 *   P:605-612 over the link census P:602, Eq. 3 PreservedBW P:714-716) and
 *   return the policy's argmax (Greedy P:777, Preserve Alg. 1)
 *   under SPEC's tie-break: lex-smallest sorted device tuple, then
 *   lex-smallest sorted used-edge list.  The reported mapping
 *   is the lex-first mapping of the winning (device set, edge set) match.
 *
 * Two enumeration modes (flags):
 *   default        canonical: one leaf per Aut(P)-orbit (lex-leader symmetry
 *                  breaking) = SPEC's deduplicated matches;
 *                  leaves scored = distinct matches = P(|F|,k)/|Aut(P)|.
 *   MAPA_F_RAW     every injective map is scored; leaves = P(|F|,k).
 * Both modes return the identical decision.
 *
 * MAPA_F_PRUNE (single-query entry points, k >= 4):
 *   branch-and-bound argmax.  A k-2 scan (the leaves sharing a prefix of k-2
 *   vertices) is skipped when an upper bound of its scores is below the best
 *   score found so far by any lane of the launch (shared through the record's
 *   `reserved` word).  The bound is exact (Eq. 1 / Eq. 3: max table entry +
 *   max column entry; Eq. 2: max rank reachable from the census by the edges
 *   the scan adds) and the test strict, so the decision is identical to the
 *   exhaustive one; only leaves_scored changes (raw_embeddings and
 *   distinct_matches are then the closed forms P(|F|,k) and P(|F|,k)/|Aut|).
 *   For k < 4 the flag is ignored.  The deep path (mapa_launch_query_wide,
 *   mapa_allocate with k > 8 or N > 32) has its own exact bounds per DFS node
 *   and work-item prefix (Greedy, Preserve-sensitive), a set search
 *   (Preserve-insensitive) and a no-enumeration Baseline; see there.
 *
 * Memory: every device pointer is caller-owned (e.g. a torch CUDA tensor);
 * streams are cudaStream_t passed as void*.  Device-side entry points are
 * asynchronous on that stream and never synchronise.
 *
 * Threads and devices: a topology or pattern handle is immutable as far as
 * the method goes, but it carries launch caches (device table images, deep
 * launch plans, CUDA graphs, staging buffers, streams) that the launch entry
 * points fill: a handle must not be used by two threads at once (the caller
 * serialises).  Patterns may be used on any device (their device
 * tables are kept per device).  A topology's mapa_allocate /
 * mapa_launch_queries state lives on the device current at its first use;
 * calling them on another device returns INVALID_ARG (load one handle per
 * device, as one process per GPU does).
 */
#ifndef MAPA_H
#define MAPA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t mapa_status;
#define MAPA_OK 0
#define MAPA_NO_CAPACITY 1      /* signal, not an error: |F| < k */
#define MAPA_E_INVALID_ARG (-1)
#define MAPA_E_PARSE (-2)       /* topology text: message names line/field */
#define MAPA_E_ALREADY_BUSY (-3) /* claim of a busy device, state unchanged */
#define MAPA_E_NOT_BUSY (-4)    /* release of a free device */
#define MAPA_E_ID_RANGE (-5)    /* device id out of range */
#define MAPA_E_UNSUPPORTED (-6) /* N > 64, k > 16; narrow-only entry points: N > 32, k > 8 or 15+W+C(k,2) > 63 */
#define MAPA_E_CUDA (-7)        /* CUDA runtime error (message has the CUDA string) */
#define MAPA_E_DISCONNECTED (-8) /* disconnected pattern, k > 1 */
#define MAPA_E_INTERNAL (-10)   /* self-check failed (decoded key inconsistent) */

/* Selectors (P:777 Greedy; Alg. 1 P:681-706 Preserve; P:777 Baseline).
 * MAPA_SEL_TOPO (trace replay / simulation only): the paper's Topo-aware
 * baseline, "recursive bi-partitioning ... under the same PCIe tree (CPU
 * socket)" (SPEC select_topo_aware S:337-344): the k lowest free
 * ids of the smallest partition with >= k free devices, where the partitions
 * are the socket groups of the topology recursively halved (by sorted id,
 * first half = ceil(n/2)), ties to the partition with the lowest device id;
 * no fitting partition -> the k lowest free ids (reading A21).  Its
 * mapping is Baseline's: the lex-smallest used-edge list on that set. */
enum { MAPA_SEL_GREEDY = 0, MAPA_SEL_PRESERVE = 1, MAPA_SEL_BASELINE = 2, MAPA_SEL_TOPO = 3 };

/* Flags. */
enum {
    MAPA_F_COMMIT = 1,              /* mapa_allocate: mark the chosen devices busy (§3.6) */
    MAPA_F_RAW = 2,                 /* score every injective map (no symmetry breaking) */
    MAPA_F_ALLOW_DISCONNECTED = 4,  /* mapa_load_pattern: accept disconnected patterns */
    MAPA_F_PRUNE = 8,               /* single query: branch-and-bound argmax (same decision) */
    MAPA_F_DEEP = 16,               /* mapa_allocate: use the deep (wide-key) kernel even when the
                                       narrow 63-bit key fits (testing / comparison) */
    MAPA_F_ZEROED = 32              /* mapa_launch_query(_wide): the caller has zeroed d_record on the
                                       stream already (e.g. one memset for several records): no
                                       per-launch memset node */
};

/* Limits.  Narrow path (mapa_launch_query, batches, traces, simulation):
 * N <= 32, k <= 8 and 15 + W + C(k,2) <= 63.  Deep path
 * (mapa_launch_query_wide): N <= 64, k <= 16. */
#define MAPA_MAX_K 16
#define MAPA_MAX_EDGES 120

/* Pattern shapes of Fig. 4 as constructed by SPEC make_pattern. */
enum { MAPA_SHAPE_RING = 0, MAPA_SHAPE_TREE = 1, MAPA_SHAPE_RINGTREE = 2,
       MAPA_SHAPE_FULL = 3, MAPA_SHAPE_EDGELESS = 4 };

typedef struct mapa_topology mapa_topology; /* immutable graph + mutable busy mask */
typedef struct mapa_pattern mapa_pattern;   /* immutable compiled pattern descriptor */

/* A decision (SPEC AllocationDecision S:322-325), host memory. */
typedef struct {
    int32_t status;          /* MAPA_OK or MAPA_NO_CAPACITY */
    int32_t k;               /* pattern vertices */
    uint64_t device_mask;    /* bit d = device d allocated */
    int8_t mapping[16];      /* mapping[i] = device of pattern vertex i (lex-first of the match) */
    int32_t m;               /* pattern edges */
    int32_t used[120][2];    /* sorted used edges (lo, hi) = E(P) ∩ E(M) realised */
    int32_t x, y, z;         /* link census: double / single(25|20) / PCIe used edges */
    int32_t agg_bw;          /* Eq. 1, GB/s */
    int32_t preserved_bw;    /* Eq. 3, GB/s */
    int32_t score;           /* selector score as packed in the key (AggBW, Eq. 2 rank, PreservedBW, 0) */
    double pred_effbw;       /* Eq. 2, double */
    uint64_t raw_embeddings;   /* P(|F|,k) injective maps (counted in RAW mode) */
    uint64_t distinct_matches; /* P(|F|,k)/|Aut(P)| (counted in canonical mode) */
    uint64_t leaves_scored;    /* leaves the kernel actually scored */
    uint64_t key;            /* narrow path: packed argmax key (mapa_record); deep path: the score word */
    uint64_t ecode[2];       /* deep path: 128-bit edge code {high, low} (0 on the narrow path) */
} mapa_decision;

/* Device-side query, 16 bytes (coalesced uint4 load). */
typedef struct {
    uint32_t busy;       /* bit d = device d busy */
    uint32_t pattern;    /* index into the pattern array of the call */
    int32_t selector;    /* MAPA_SEL_* */
    int32_t sensitive;   /* PRESERVE: 1 = bandwidth sensitive (Alg. 1) */
} mapa_query;

/* Device-side query of the deep path, 16 bytes (N <= 64). */
typedef struct {
    uint64_t busy;       /* bit d = device d busy */
    int32_t selector;    /* ignored by the launch (the call's selector decides) */
    int32_t sensitive;
} mapa_query64;

/* Device-side result record, 32 bytes.
 *   key = score << (W + C(k,2)) | brev_W(S) << C(k,2) | ecode, where W is the
 *   topology width (8/16/32), brev_W(S) sets bit W-1-d for every chosen
 *   device d (larger = lex-smaller device tuple) and ecode sets bit
 *   C(k,2)-1-p for every used edge whose endpoint ranks inside S form the
 *   p-th pair in lex order (larger = lex-smaller used-edge list).  key 0 =
 *   no match (no capacity).  Max over keys = the policy's choice. */
typedef struct {
    uint64_t key;
    uint64_t leaves;     /* leaves scored */
    uint32_t ctr;        /* work-item counter (scratch, zeroed by the launch) */
    uint32_t status;     /* 0 ok; nonzero = the launch refused the query and scored nothing:
                            1 = the 16-bit scan's range does not fit this free set (a busy_hint
                            that lied: see mapa_launch_query), 2 = the single-query kernel's
                            static shared tables are not at the window address its code
                            addresses them by (never seen; a guard, not a mode) -- mapa_decode
                            reports MAPA_E_INVALID_ARG for both */
    uint64_t reserved;   /* scratch (MAPA_F_PRUNE: best score + 1 found so far), zeroed by the launch */
} mapa_record;

/* Deep-path result record, 64 bytes (k <= 16, N <= 64; SURVEY §8(f) NEXT 1
 * and NEXT 4).  The argmax key is 256 bits, compared lexicographically as
 * (score, set, ecode_hi, ecode_lo):
 *   score = the selector score (AggBW, Eq. 2 rank, PreservedBW, 0)
 *   set   = brev_64(S): bit 63-d set for every chosen device d (larger =
 *           lex-smaller device tuple)
 *   ecode = 128-bit edge code: bit C(k,2)-1-p set for every used edge whose
 *           endpoint ranks inside S form the p-th pair in lex order (larger =
 *           lex-smaller used-edge list); ecode_hi holds bits 64..127.
 * set 0 = no match.  The launch zeroes the record; `lock` serialises the
 * per-CTA merges of the maximum (order independent, so the result is
 * deterministic for every grid size and rank count). */
typedef struct {
    uint64_t score;
    uint64_t set;
    uint64_t ecode_hi;
    uint64_t ecode_lo;
    uint64_t leaves;     /* leaves scored */
    uint32_t ctr;        /* work-item counter (scratch) */
    uint32_t lock;       /* merge lock (scratch) */
    uint32_t status;     /* 0 ok; nonzero = device-side argument error */
    uint32_t pad;
    uint64_t reserved;   /* scratch: running max of (score << 32 | set >> 32): merge filter, branch-and-bound incumbent */
} mapa_wide_record;

/* Trace op (C2 replay): op 0 = ALLOC job, 1 = RELEASE job. */
typedef struct {
    int32_t op;
    int32_t job;
} mapa_trace_op;

/* ---------------------------------------------------------------- topology */

/* Builtin name (dgx1v, dgx1p, summit, torus2d16, cubemesh16: S:43-51,
 * S:105-110) when is_text == 0, else the topology text format of DESIGN.md
 * (fields of S:115: name, devices, sockets, link a b class; 1-based ids;
 * unlisted pairs are PCIe).  N <= 64; topologies with N > 32 run on the
 * deep path only (bigger servers).  *out owned by the caller,
 * freed with mapa_free_topology.  Errors: PARSE (message names the line),
 * ID_RANGE, UNSUPPORTED (N > 64), INVALID_ARG. */
mapa_status mapa_load_topology(const char *builtin_or_text, int32_t is_text, mapa_topology **out);
void mapa_free_topology(mapa_topology *t);

/* N, padded width W (8, 16, 32 or 64), link bandwidth matrix bw[N*N] (GB/s,
 * diagonal 0; may be NULL) and the busy mask. */
mapa_status mapa_topology_info(const mapa_topology *t, int32_t *n, int32_t *width, int32_t *bw,
                               uint64_t *busy);

/* State management (§3.6; SPEC allocate_devices S:70-78,
 * release_devices S:79-87).  claim: ALREADY_BUSY / ID_RANGE with state
 * unchanged; release: NOT_BUSY / ID_RANGE. set_busy replaces the mask
 * (checkpoint/restore). */
mapa_status mapa_claim(mapa_topology *t, uint64_t device_mask);
mapa_status mapa_release(mapa_topology *t, uint64_t device_mask);
mapa_status mapa_set_busy(mapa_topology *t, uint64_t busy);

/* ---------------------------------------------------------------- patterns */

/* Pattern from an edge list (2*m ints, 0-based vertex ids < k).  1 <= k <= 16,
 * 0 <= m <= C(k,2).  Duplicate edges and self loops: INVALID_ARG.
 * Disconnected with k > 1: DISCONNECTED unless MAPA_F_ALLOW_DISCONNECTED
 * (S:210).  Compiles the point-stabiliser chain of Aut(P) (backtracking:
 * orbit of i under the automorphisms fixing 0..i-1), |Aut(P)| = product of
 * the orbit sizes, the lex-leader symmetry constraints and the Eq. 2 rank
 * table for m.  Patterns with k > 8 (or a key wider than 63 bits on the
 * topology) run on the deep path only. */
mapa_status mapa_load_pattern(int32_t k, int32_t m, const int32_t *edges, uint32_t flags,
                              mapa_pattern **out);
/* SPEC make_pattern: Ring (k=2: one edge; k=1: INVALID_ARG),
 * Tree (children of i are 2i+1, 2i+2), RingTree (union), Full, Edgeless. */
mapa_status mapa_make_pattern(int32_t shape, int32_t k, mapa_pattern **out);
void mapa_free_pattern(mapa_pattern *p);

typedef struct {
    int32_t k, m;
    int32_t aut_order;       /* |Aut(P)|, clamped to INT32_MAX (aut_order64 is exact) */
    uint16_t back[16];       /* back[j] bit i: edge (i,j), i < j */
    uint16_t lex_src[16];    /* lex_src[u] bit i: canonical mode requires f(i) < f(u) */
    int32_t edges[120][2];   /* normalised (a<b), sorted */
    uint64_t aut_order64;    /* |Aut(P)| (16! fits) */
} mapa_pattern_info;
mapa_status mapa_get_pattern_info(const mapa_pattern *p, mapa_pattern_info *out);

/* Eq. 2 with Table 4 theta, double. */
double mapa_pred_effbw(int32_t x, int32_t y, int32_t z);
/* Dense rank of Eq. 2 over the censuses with x+y+z = m: out[x*(m+1)+y]
 * (entries with x+y > m are 0).  m <= 120 (reading A9: no ties, double order
 * = exact order for every m <= 120). */
mapa_status mapa_effbw_rank_table(int32_t m, uint16_t *out);

/* Eq. 2 with any 14 coefficients (theta NULL = Table 4). */
double mapa_pred_effbw_theta(const double *theta, int32_t x, int32_t y, int32_t z);

/* fit_effbw_model (§3.4.3 "non-linear polynomial regression",
 * P:614-616): ordinary least squares of Eq. 2's 14 features (linear in
 * theta) over n samples census[3n] = (x, y, z), bw[n] GB/s, by Householder QR.
 * theta[14] out; diag[4] (may be NULL) = relative error ||r|| / ||bw||, RMSE,
 * MAE, condition estimate max|R_jj| / min|R_jj| (reading A23).
 * Errors: INVALID_ARG for n < 14 or a rank-deficient feature matrix (the
 * message names the dependent feature). */
mapa_status mapa_fit_effbw(int32_t n, const int32_t *census, const double *bw, double *theta, double *diag);

/* Replace the pattern's Eq. 2 model (default Table 4): rebuilds its rank
 * table; decisions and reported pred_effbw of this pattern use theta.  Not
 * safe while a launch with this pattern is being prepared on another thread. */
mapa_status mapa_pattern_set_effbw_model(mapa_pattern *p, const double *theta);

/* ---------------------------------------------------------- single query */

/* One allocation end to end, host buffers: stages the query (16 B) to the
 * device from pinned memory, launches the enumerate-score-argmax kernel on
 * cuda_stream (NULL = default stream) -- the narrow kernel when the 63-bit key
 * fits and MAPA_F_DEEP is not set, else the deep kernel
 * (mapa_launch_query_wide) -- reads the record back, decodes it
 * on the host and, with MAPA_F_COMMIT, marks the devices busy.  Blocks until
 * the stream reaches the copy.  Returns MAPA_OK, MAPA_NO_CAPACITY (out->status
 * too) or an error. Not thread-safe per topology handle. */
mapa_status mapa_allocate(mapa_topology *t, const mapa_pattern *p, int32_t selector,
                          int32_t bw_sensitive, uint32_t flags, void *cuda_stream,
                          mapa_decision *out);

/* nq (1..32) independent allocations on the topology's current busy mask,
 * end to end from host buffers in ONE call: one H2D copy stages every query
 * (and zeroes every device record), the nq enumerate-score-argmax launches
 * run as parallel branches of one cached CUDA graph (their prologues and
 * tails overlap), one D2H copy brings the records back, and each is decoded
 * on the host exactly as mapa_allocate would (pats[i], selector[i],
 * sensitive[i]; narrow or deep path per query).  Never commits
 * (MAPA_F_COMMIT: INVALID_ARG): the queries see the same state.  out[nq]; a
 * query without capacity gets status MAPA_NO_CAPACITY in its decision.
 * Blocks until the stream reaches the copy.  Errors as mapa_allocate. */
mapa_status mapa_allocate_many(mapa_topology *t, const mapa_pattern *const *pats, int32_t nq, const int32_t *selector,
                               const int32_t *sensitive, uint32_t flags, void *cuda_stream, mapa_decision *out);

/* Device-resident launch of one query's shard: zeroes d_record (unless
 * MAPA_F_ZEROED: the caller zeroed it on cuda_stream) and
 * enumerates the work items i with i % world == rank of the query whose busy
 * mask is read from d_query->busy on the device (the other d_query fields are
 * ignored; p, selector and sensitive choose the kernel).  rank = 0, world = 1
 * for the whole query.  Asynchronous on cuda_stream.  Records of the R shards
 * combine by max(key), sum(leaves) (mapa_reduce_records or an NCCL
 * MAX/SUM all-reduce), then mapa_decode gives the same decision for every R
 * (S:369).  busy_hint: the busy mask if the host knows it (sizes the grid),
 * else 0xFFFFFFFF. */
mapa_status mapa_launch_query(const mapa_topology *t, const mapa_pattern *p, int32_t selector,
                              int32_t sensitive, const mapa_query *d_query, mapa_record *d_record,
                              uint32_t flags, int32_t rank, int32_t world, uint64_t busy_hint,
                              void *cuda_stream);

/* nq independent single queries (narrow path) from ONE call: zeroes
 * d_records[nq] once, forks `nstreams` internal streams (owned by the
 * topology, created on first use) from cuda_stream with an event and makes
 * cuda_stream wait for all of them: ordered like one launch on cuda_stream.
 * Queries that score fewer than 2^22 leaves (P(|F|,k), /|Aut| canonical) run
 * together in ONE batch launch (the mapa_allocate_batch kernel over a
 * host-built order of those queries, grouped by (k, selector)) on the first
 * stream, when every pattern fits the batch kernel (npats <= 16, k <= 8) and
 * MAPA_F_PRUNE is not set; every other query gets a full-GPU mapa_launch_query
 * (its busy mask from h_queries[i] plans the grid; the kernel reads
 * d_queries[i]) round-robin over the streams.  The records are the same
 * either way.  pats[npats] indexed by the query's `pattern`.  Errors as
 * mapa_launch_query (the first failing query's; earlier launches stay
 * enqueued). */
mapa_status mapa_launch_queries(mapa_topology *t, const mapa_pattern *const *pats, int32_t npats, int32_t nq,
                                const mapa_query *h_queries, const mapa_query *d_queries, mapa_record *d_records,
                                uint32_t flags, int32_t nstreams, void *cuda_stream);

/* Host: combine n shard records (max key, sum leaves). */
mapa_status mapa_reduce_records(const mapa_record *records, int32_t n, mapa_record *out);

/* Host: decode a (combined) record into a decision for (busy, selector,
 * sensitive, flags).  Recomputes census, AggBW, PreservedBW and Eq. 2 from
 * the decoded (S, mapping) and checks them against the key's score. */
mapa_status mapa_decode(const mapa_topology *t, const mapa_pattern *p, uint64_t busy,
                        int32_t selector, int32_t bw_sensitive, uint32_t flags,
                        const mapa_record *record, mapa_decision *out);

/* ------------------------------------------------- deep patterns (k <= 16) */

/* Device-resident launch of one query's shard on the deep path (SURVEY §8(f)
 * NEXT 1: the paper's overhead study reaches "9 GPUs and above" on 16-GPU
 * graphs).  Same contract as mapa_launch_query (busy read from
 * d_query->busy on the device; work item i of the prefix space goes to rank
 * i's stripe owner; asynchronous on cuda_stream) but with the 256-bit key of
 * mapa_wide_record, so any k <= 16 on any N <= 64 fits.  Enumeration: a
 * warp-uniform explicit-stack DFS over the first k-L pattern vertices, then
 * the last L vertices (L = 1..4, chosen on the host) as a lane-parallel scan
 * over a table of index tuples into the remaining free devices.  RAW and
 * canonical modes as for the narrow path.  MAPA_F_PRUNE (Greedy, and
 * Preserve-sensitive when (k+1)(m+1)^2 <= 17408; other selectors ignore it
 * here): branch and bound with exact bounds.  Greedy (Eq. 1) -- a
 * prefix subtree is skipped when its score so far plus, for every pattern edge
 * from a placed vertex into the unplaced part, the best free link of that
 * vertex's device, plus (edges inside the unplaced part) x (best free pair) is
 * below the best score published by any lane (the record's reserved word); a
 * node's suffix scan is skipped when the sum of its tables' maxima is below it.
 * Preserve-sensitive (Eq. 2): after nd placed vertices with census (x0, y0)
 * and c edges still unplaced, the bound is max rank over (x0+a, y0+b), a+b <=
 * c (host tables uploaded with the rank table).  On a score tie the subtree
 * is still cut when U + the lowest k-nd other free devices orders below the
 * published best set (the reserved word holds score << 32 | brev64(S) >> 32).
 * mapa_allocate with MAPA_F_PRUNE and Preserve-insensitive on the deep path
 * searches device SETS instead (Eq. 3 depends on the set only): the full-k
 * pattern's decision gives the set, the pattern's lex-smallest labelling
 * (weight independent, cached per pattern) gives the edges; exact.  Baseline
 * with MAPA_F_PRUNE on the deep path: the k lowest free ids and that
 * labelling, no enumeration (leaves_scored 0).
 * Strict tests: the decision equals the exhaustive one; leaves counts what was
 * scored (the decision's raw / distinct are then the closed forms).
 * Errors: INVALID_ARG, UNSUPPORTED (k > 16), CUDA. */
mapa_status mapa_launch_query_wide(const mapa_topology *t, const mapa_pattern *p, int32_t selector,
                                   int32_t sensitive, const mapa_query64 *d_query, mapa_wide_record *d_record,
                                   uint32_t flags, int32_t rank, int32_t world, uint64_t busy_hint,
                                   void *cuda_stream);

/* Host: combine n deep shard records (lexicographic max of the 256-bit key,
 * sum of leaves, OR of status). */
mapa_status mapa_reduce_wide_records(const mapa_wide_record *records, int32_t n, mapa_wide_record *out);

/* Host: decode a (combined) deep record.  The lex-first mapping of the
 * winning (device set, edge set) is found by backtracking in pattern-vertex
 * order over the devices of S in ascending order, keeping only partial maps
 * whose placed pattern edges land on decoded edges (first complete map =
 * lex-first).  Scores are recomputed and checked against the key. */
mapa_status mapa_decode_wide(const mapa_topology *t, const mapa_pattern *p, uint64_t busy,
                             int32_t selector, int32_t bw_sensitive, uint32_t flags,
                             const mapa_wide_record *record, mapa_decision *out);

/* ---------------------------------------------------------------- batches */

/* nq independent queries (never committed; each carries its own busy mask),
 * d_queries[nq] -> d_results[nq] records.  pats[npats] (npats <= 16, every
 * pattern k <= 8 and sum of (m+1)^2 rank-table entries <= 4096).
 * d_scratch: >= 512 + 4*nq bytes of device memory (work counter, and the
 * query order: with more than one pattern, queries are bucketed by code path
 * -- (k, selector) -- with a device counting sort before the batch kernel, so
 * consecutive warps run the same kernel instantiation; results do not depend
 * on the order).
 * Asynchronous on cuda_stream.  A query with a bad pattern index or an
 * unsupported key budget gets record.status = 1 and key 0. */
mapa_status mapa_allocate_batch(const mapa_topology *t, const mapa_pattern *const *pats,
                                int32_t npats, int64_t nq, const mapa_query *d_queries,
                                mapa_record *d_results, void *d_scratch, uint32_t flags,
                                void *cuda_stream);

/* Host: deal nq independent queries (host copies, as for the batch) over
 * `world` ranks for a multi-GPU batch (batches shard by query,
 * no data-path collective).  A query's work is the number of leaves its launch
 * scores, P(|F|,k) with MAPA_F_RAW, else P(|F|,k)/|Aut(P)| (0 without
 * capacity); queries are taken heaviest first (ties by index) and each goes
 * to the least-loaded rank (ties by rank): longest-processing-time-first,
 * deterministic, every rank's load <= mean + the largest query.  owner[nq]
 * out (rank of each query); load[world] (may be NULL) out, in leaves.
 * Errors: INVALID_ARG (a pattern index out of range). */
mapa_status mapa_shard_queries(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats, int64_t nq,
                               const mapa_query *queries, uint32_t flags, int32_t world, int32_t *owner,
                               double *load);

/* ----------------------------------------------------------- trace replay */

/* C2: ntraces independent FIFO traces replayed entirely on the device, one
 * CTA per trace.  Trace t has nops ops d_ops[t*nops ...] and njobs jobs
 * d_jobs[t*njobs ...] (mapa_query with busy ignored, pattern/selector/
 * sensitive per job).  ALLOC j: the kernel enumerates, scores and selects on
 * the trace's current busy mask, stores the winning key in
 * d_keys[t*njobs + j] and marks the devices busy; RELEASE j frees them
 * (§3.6).  An ALLOC without capacity stores key 0 and leaves the state.
 * Asynchronous. */
mapa_status mapa_trace_replay(const mapa_topology *t, const mapa_pattern *const *pats,
                              int32_t npats, int32_t ntraces, int32_t nops,
                              const mapa_trace_op *d_ops, int32_t njobs, const mapa_query *d_jobs,
                              uint64_t *d_keys, uint32_t flags, void *cuda_stream);

/* Host: decode ONE replayed trace (its njobs keys from mapa_trace_replay,
 * copied to host memory) into full decisions out[njobs] (job order).  The op
 * order is replayed on the host (§3.6 state management): ALLOC j
 * decodes keys[j] against the busy mask of that moment -- device set, lex-first
 * mapping, used edges, census, Eq. 1 / 2 / 3 recomputed and checked against the
 * key's score, as mapa_decode -- then marks its devices busy; RELEASE j frees
 * them.  jobs[njobs] = the host copy of the mapa_query array the replay used
 * (pattern / selector / sensitive per job; MAPA_SEL_TOPO decodes as Baseline,
 * reading A21).  The trace kernel counts no leaves, so raw_embeddings and
 * distinct_matches are the closed forms P(|F|,k) and P(|F|,k)/|Aut| and
 * leaves_scored is 0.  A key of 0, or a job without an ALLOC op, gives status
 * MAPA_NO_CAPACITY in its decision (the call itself returns MAPA_OK).  Errors:
 * INVALID_ARG (index out of range, a job allocated twice), INTERNAL (a key that
 * overlaps the busy devices or contradicts its score), outputs untouched. */
mapa_status mapa_decode_trace(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats,
                              int32_t nops, const mapa_trace_op *ops, int32_t njobs, const mapa_query *jobs,
                              const uint64_t *keys, uint32_t flags, mapa_decision *out);

/* ------------------------------------------------------------- simulator */

/* One job of a simulated stream (SPEC JobSpec / run_simulation, S:386-439;
 * the execution framework of Fig. 13). */
typedef struct {
    int32_t pattern;     /* index into the pattern array of the call */
    int32_t sensitive;   /* bandwidth sensitive (Preserve's Alg. 1 branch) */
    double duration;     /* simulated seconds, allocation independent */
    double arrival;      /* simulated seconds (0 = the paper's batch at t = 0) */
} mapa_job;

/* Policies of the paper's evaluation (§4; SPEC policy names). */
enum { MAPA_POLICY_BASELINE = 0, MAPA_POLICY_TOPO = 1, MAPA_POLICY_GREEDY = 2, MAPA_POLICY_PRESERVE = 3 };

/* SPEC JobLogRecord: the allocation of one job and its times. */
typedef struct {
    int32_t job, k;
    uint32_t device_mask;
    int32_t x, y, z;           /* link census of the used edges */
    int32_t agg_bw;            /* Eq. 1 */
    int32_t preserved_bw;      /* Eq. 3 on the free set at allocation time */
    double pred_effbw;         /* Eq. 2 */
    double arrival, start, end, wait;  /* simulated seconds; wait = start - arrival */
} mapa_job_log;

/* Strict-FIFO event schedule: the head job starts as soon as it
 * has arrived and |F| >= k; finish events at equal times are processed before
 * allocation attempts, in job order.  Because the hardware graph is complete
 * and durations are allocation independent, the schedule depends only
 * on the free COUNT, hence not on the policy.  Outputs (caller-owned host
 * arrays): ops[2*njobs] = (op, job) with op 0 = ALLOC, 1 = RELEASE, and
 * start[njobs], end[njobs].  Errors: INVALID_ARG (a job larger than the
 * machine; negative duration / arrival). */
mapa_status mapa_fifo_schedule(int32_t n_devices, int32_t njobs, const int32_t *k, const double *duration,
                               const double *arrival, mapa_trace_op *ops, double *start, double *end);

/* run_simulation: schedule the jobs, replay the allocations of
 * `policy` on the device (one CTA, mapa_trace_replay's kernel: Topo-aware /
 * Baseline / Greedy / Preserve decided and committed per ALLOC in shared
 * memory), then decode every decision on the host into out[njobs] (job
 * order).  The topology's own busy mask is not used or changed (the
 * simulation starts idle).  Patterns must fit the narrow path (k <= 8).
 * Blocks until done.  Errors: INVALID_ARG, UNSUPPORTED, CUDA, INTERNAL. */
mapa_status mapa_simulate(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats, int32_t njobs,
                          const mapa_job *jobs, int32_t policy, uint32_t flags, void *cuda_stream,
                          mapa_job_log *out);

/* summarize_log quantiles: min, 25th, 50th, 75th percentile, max
 * of v[n] by linear interpolation between order statistics ("type 7":
 * position p*(n-1)).  out[5].  Errors: INVALID_ARG for n < 1. */
mapa_status mapa_quantiles(const double *v, int32_t n, double *out);

/* Thread-local message of the last failing call on this thread. */
const char *mapa_last_error(void);
/* Library version string. */
const char *mapa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MAPA_H */
