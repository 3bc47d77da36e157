/*
 * MAPA CPU oracle in plain C -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with the
 * CUDA path (paper_2110_03214_b200/csrc): it is the same plain definition as
 * oracle/mapa_oracle.py, written in C so that the large configurations finish.
 *
 * Definition followed (PAPER.md / SPEC.md citations):
 *   - matches: every injective map V(P)->F is an embedding because the hardware
 *     graph is complete; matches are deduplicated by
 *     (device set, used-edge set) (reading A2);
 *   - Eq. 1 AggBW = sum of w over used edges;
 *   - census (x,y,z) over used edges, 25 and 20 both count toward y
 *     (reading A5);
 *   - Eq. 2 predicted EffBW with Table 4 theta, double;
 *   - Eq. 3 PreservedBW = sum of w over pairs of free devices not in S
 *     (reading A6), direct double loop;
 *   - selection: strict '>' over matches in lex order of (sorted device tuple,
 *     sorted used-edge list) = Alg. 1 first-wins loop + SPEC tie-break
 *     (SPEC S:349).
 *
 * Parallelism: pthreads over the index a of the first device S[0] = F[a] of
 * each lexicographic k-subset; per-a results are combined in increasing a,
 * strict '>', so the result is identical for every thread count.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t status;        /* 0 ok, 1 no capacity, <0 error */
    int32_t k;
    uint32_t device_mask;  /* bit d = device d (0-based) */
    int8_t mapping[8];     /* mapping[i] = device of pattern vertex i */
    int32_t m;
    int32_t used[28][2];   /* sorted used edges (lo, hi) */
    int32_t x, y, z, agg_bw, preserved_bw;
    int32_t pad;
    double pred_effbw;
    double score;
    uint64_t raw, distinct;
} oracle_result;

/* Table 4 */
static const double THETA[14] = {16.396, 4.536, 1.556, -20.694, -9.467, 7.615, -7.973,
                                 12.733, -4.195, -8.413, 62.851, 27.418, -5.114, -46.973};

double oracle_eq2(int x, int y, int z) {
    const double *t = THETA;
    double X = x, Y = y, Z = z;
    return t[0] * X + t[1] * Y + t[2] * Z + t[3] / (X + 1) + t[4] / (Y + 1) + t[5] / (Z + 1) +
           t[6] * X * Y + t[7] * Y * Z + t[8] * Z * X + t[9] / (X * Y + 1) + t[10] / (Y * Z + 1) +
           t[11] / (Z * X + 1) + t[12] * X * Y * Z + t[13] / (X * Y * Z + 1);
}

typedef struct {
    int n, k, m, selector, sensitive;
    const int32_t *w;     /* n*n weights */
    const int32_t *pe;    /* 2m pattern edges */
    int nf;
    int F[64];
} ctx_t;

typedef struct {
    int found;
    double score;
    int S[8];
    int pi[8];
    int E[28][2];
    int agg, x, y, z, pres;
    double eff;
    uint64_t raw, distinct;
} unit_t;

typedef struct {
    uint16_t code[28];
    int8_t pi[8];
    int32_t idx;
    int m;
} entry_t;

static int cmp_entry(const void *a, const void *b) {
    const entry_t *p = (const entry_t *)a, *q = (const entry_t *)b;
    for (int i = 0; i < p->m; i++) {
        if (p->code[i] != q->code[i]) return p->code[i] < q->code[i] ? -1 : 1;
    }
    return p->idx < q->idx ? -1 : (p->idx > q->idx);
}

/* std::next_permutation on a small int array; returns 0 after the last. */
static int next_perm(int *a, int n) {
    int i = n - 2;
    while (i >= 0 && a[i] >= a[i + 1]) i--;
    if (i < 0) return 0;
    int j = n - 1;
    while (a[j] <= a[i]) j--;
    int t = a[i]; a[i] = a[j]; a[j] = t;
    for (int l = i + 1, r = n - 1; l < r; l++, r--) { t = a[l]; a[l] = a[r]; a[r] = t; }
    return 1;
}

static void score_match(const ctx_t *c, const int *S, const entry_t *e, unit_t *u) {
    int n = c->n;
    int agg = 0, x = 0, y = 0, z = 0;
    for (int i = 0; i < c->m; i++) {
        int lo = e->code[i] >> 6, hi = e->code[i] & 63;
        int b = c->w[lo * n + hi];
        agg += b;                                   /* Eq. 1 */
        if (b == 50) x++;                           /* census */
        else if (b == 25 || b == 20) y++;
        else z++;
    }
    double eff = oracle_eq2(x, y, z);               /* Eq. 2 */
    int inS[64] = {0};
    for (int i = 0; i < c->k; i++) inS[S[i]] = 1;
    int pres = 0;                                   /* Eq. 3 */
    for (int i = 0; i < c->nf; i++) {
        if (inS[c->F[i]]) continue;
        for (int j = i + 1; j < c->nf; j++) {
            if (inS[c->F[j]]) continue;
            pres += c->w[c->F[i] * n + c->F[j]];
        }
    }
    double s;
    if (c->selector == 0) s = agg;
    else if (c->selector == 1) s = c->sensitive ? eff : pres;
    else s = 0.0;
    if (!u->found || s > u->score) {
        u->found = 1;
        u->score = s;
        for (int i = 0; i < c->k; i++) { u->S[i] = S[i]; u->pi[i] = e->pi[i]; }
        for (int i = 0; i < c->m; i++) { u->E[i][0] = e->code[i] >> 6; u->E[i][1] = e->code[i] & 63; }
        u->agg = agg; u->x = x; u->y = y; u->z = z; u->pres = pres; u->eff = eff;
    }
}

static void process_subset(const ctx_t *c, const int *S, entry_t *ent, unit_t *u) {
    int k = c->k, m = c->m;
    int perm[8];
    memcpy(perm, S, sizeof(int) * k);
    int cnt = 0;
    do {                                            /* permutations in lex order */
        u->raw++;
        entry_t *e = &ent[cnt];
        e->m = m;
        e->idx = cnt;
        for (int i = 0; i < k; i++) e->pi[i] = (int8_t)perm[i];
        for (int i = 0; i < m; i++) {
            int a = perm[c->pe[2 * i]], b = perm[c->pe[2 * i + 1]];
            int lo = a < b ? a : b, hi = a < b ? b : a;
            uint16_t code = (uint16_t)(lo * 64 + hi);
            int j = i;                              /* insertion sort */
            while (j > 0 && e->code[j - 1] > code) { e->code[j] = e->code[j - 1]; j--; }
            e->code[j] = code;
        }
        cnt++;
    } while (next_perm(perm, k));
    qsort(ent, cnt, sizeof(entry_t), cmp_entry);    /* sorted(seen), first pi kept */
    for (int i = 0; i < cnt; i++) {
        if (i > 0 && memcmp(ent[i].code, ent[i - 1].code, sizeof(uint16_t) * m) == 0) continue;
        u->distinct++;
        score_match(c, S, &ent[i], u);
    }
}

/* One work unit = every k-subset whose first two elements are F[a], F[b]
 * (b < 0 when k == 1: the single subset {F[a]}), in lex order. */
static void process_unit(const ctx_t *c, int a, int b, entry_t *ent, unit_t *u) {
    memset(u, 0, sizeof(*u));
    int k = c->k, nf = c->nf;
    int idx[8];
    int S[8];
    idx[0] = a;
    if (k > 1) {
        idx[1] = b;
        for (int i = 2; i < k; i++) idx[i] = b + i - 1;
    }
    if (idx[k - 1] >= nf) return;
    for (;;) {
        for (int i = 0; i < k; i++) S[i] = c->F[idx[i]];
        process_subset(c, S, ent, u);
        int i = k - 1;                              /* next combination, idx[0..1] fixed */
        while (i >= 2 && idx[i] == nf - k + i) i--;
        if (i < 2) break;
        idx[i]++;
        for (int j = i + 1; j < k; j++) idx[j] = idx[j - 1] + 1;
    }
}

typedef struct {
    const ctx_t *c;
    unit_t *units;
    int (*ab)[2];
    int nunits;
    int next;
    pthread_mutex_t mu;
} pool_t;

static size_t fact(int k) { size_t f = 1; for (int i = 2; i <= k; i++) f *= i; return f; }

static void *worker(void *arg) {
    pool_t *p = (pool_t *)arg;
    entry_t *ent = (entry_t *)malloc(sizeof(entry_t) * fact(p->c->k));
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int i = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (i >= p->nunits) break;
        process_unit(p->c, p->ab[i][0], p->ab[i][1], ent, &p->units[i]);
    }
    free(ent);
    return NULL;
}

/* Brute-force allocation.  w: n*n weights (GB/s, diagonal ignored); busy: bit d
 * busy; pe: 2m pattern edges (0-based); selector 0 GREEDY, 1 PRESERVE, 2 BASELINE.
 * a_lo/a_hi restrict S[0] to F[a_lo..a_hi) and b_lo/b_hi restrict S[1] to
 * F[b_lo..b_hi) (bounded samples); a negative bound = unrestricted.  Work units
 * are the (S[0], S[1]) pairs, combined in lex order, so the result does not
 * depend on the thread count.  Returns 0, or <0 on invalid arguments. */
int oracle_allocate(int n, const int32_t *w, uint32_t busy, int k, int m, const int32_t *pe,
                    int selector, int sensitive, int nthreads, int a_lo, int a_hi, int b_lo,
                    int b_hi, oracle_result *out) {
    memset(out, 0, sizeof(*out));
    if (n < 1 || n > 32 || k < 1 || k > 8 || m < 0 || m > 28) return -1;
    ctx_t c;
    c.n = n; c.k = k; c.m = m; c.selector = selector; c.sensitive = sensitive; c.w = w; c.pe = pe;
    c.nf = 0;
    for (int d = 0; d < n; d++)
        if (!((busy >> d) & 1u)) c.F[c.nf++] = d;
    out->k = k;
    out->m = m;
    if (k > c.nf) { out->status = 1; return 0; }
    int lo = a_lo < 0 ? 0 : a_lo;
    int hi = a_hi < 0 ? c.nf - k + 1 : a_hi;
    if (hi > c.nf - k + 1) hi = c.nf - k + 1;
    if (lo >= hi) { out->status = 1; return 0; }
    int bmax = c.nf - k + 2;
    int blo = b_lo < 0 ? 0 : b_lo, bhi = b_hi < 0 ? bmax : (b_hi < bmax ? b_hi : bmax);
    pool_t p;
    p.c = &c;
    p.ab = (int (*)[2])malloc(sizeof(int[2]) * (size_t)(hi - lo) * (k > 1 ? c.nf : 1));
    p.nunits = 0;
    for (int a = lo; a < hi; a++) {
        if (k == 1) { p.ab[p.nunits][0] = a; p.ab[p.nunits][1] = -1; p.nunits++; continue; }
        for (int b = (a + 1 > blo ? a + 1 : blo); b < bhi; b++) {
            p.ab[p.nunits][0] = a; p.ab[p.nunits][1] = b; p.nunits++;
        }
    }
    p.next = 0;
    p.units = (unit_t *)calloc(p.nunits > 0 ? p.nunits : 1, sizeof(unit_t));
    pthread_mutex_init(&p.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, worker, &p);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&p.mu);
    unit_t best;
    memset(&best, 0, sizeof(best));
    uint64_t raw = 0, distinct = 0;
    for (int i = 0; i < p.nunits; i++) {            /* combine in lex order, strict '>' */
        unit_t *u = &p.units[i];
        raw += u->raw;
        distinct += u->distinct;
        if (u->found && (!best.found || u->score > best.score)) best = *u;
    }
    free(p.units);
    free(p.ab);
    out->raw = raw;
    out->distinct = distinct;
    out->status = best.found ? 0 : 1;
    if (!best.found) return 0;
    out->score = best.score;
    out->device_mask = 0;
    for (int i = 0; i < k; i++) {
        out->device_mask |= 1u << best.S[i];
        out->mapping[i] = (int8_t)best.pi[i];
    }
    for (int i = 0; i < m; i++) { out->used[i][0] = best.E[i][0]; out->used[i][1] = best.E[i][1]; }
    out->x = best.x; out->y = best.y; out->z = best.z;
    out->agg_bw = best.agg; out->preserved_bw = best.pres; out->pred_effbw = best.eff;
    return 0;
}

/* ------------------------------------------------------------------------
 * Deep oracle (k <= 16).  The same definition as
 * oracle_allocate, restated without the per-subset table of edge lists (k!
 * entries per subset does not fit for k > 8):
 *   for every k-subset S of F in lex order, for every permutation pi of S in
 *   lex order: E = sorted used-edge list, score by Eq. 1 / Eq. 2 / Eq. 3;
 *   the winner is the max score; ties go to the earlier S (lex-smaller device
 *   tuple), then within S to the lex-smaller E, and for an equal (S, E) the
 *   first pi is kept (the lex-first mapping) -- SPEC S:349; Alg. 1's
 *   first-wins loop.  `distinct` is not counted here (0).
 * Work units = (subset, index of pi[0] in S), combined in that order with the
 * same rule, so the result does not depend on the thread count.
 * ------------------------------------------------------------------------ */
typedef struct {
    int32_t status, k;
    uint64_t device_mask;
    int8_t mapping[16];
    int32_t m;
    int32_t used[120][2];
    int32_t x, y, z, agg_bw, preserved_bw, pad;
    double pred_effbw, score;
    uint64_t raw;
} oracle_result_deep;

typedef struct {
    int found;
    double score;
    int S[16], pi[16];
    uint16_t E[120];
    int agg, x, y, z, pres;
    double eff;
    uint64_t raw;
} dunit_t;

typedef struct {
    const ctx_t *c;
    int (*subsets)[16];   /* lex-ordered k-subsets */
    int nsub;
    dunit_t *units;       /* nsub * k */
    int nunits, next;
    pthread_mutex_t mu;
} dpool_t;

static int cmp_codes(const uint16_t *a, const uint16_t *b, int m) {
    for (int i = 0; i < m; i++)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

static void deep_unit(const ctx_t *c, const int *S, int i0, dunit_t *u) {
    int k = c->k, m = c->m, n = c->n;
    memset(u, 0, sizeof(*u));
    int inS[64] = {0};
    for (int i = 0; i < k; i++) inS[S[i]] = 1;
    int pres = 0;                                   /* Eq. 3 (depends on S only) */
    for (int i = 0; i < c->nf; i++) {
        if (inS[c->F[i]]) continue;
        for (int j = i + 1; j < c->nf; j++) {
            if (inS[c->F[j]]) continue;
            pres += c->w[c->F[i] * n + c->F[j]];
        }
    }
    int perm[16], rest[16], nr = 0;
    for (int i = 0; i < k; i++)
        if (i != i0) rest[nr++] = S[i];
    perm[0] = S[i0];
    uint16_t E[120];
    do {                                            /* permutations with pi[0] = S[i0], lex order */
        for (int i = 0; i < nr; i++) perm[i + 1] = rest[i];
        u->raw++;
        int agg = 0, x = 0, y = 0, z = 0;
        for (int i = 0; i < m; i++) {
            int a = perm[c->pe[2 * i]], b = perm[c->pe[2 * i + 1]];
            int lo = a < b ? a : b, hi = a < b ? b : a;
            uint16_t code = (uint16_t)(lo * 64 + hi);
            int j = i;                              /* insertion sort */
            while (j > 0 && E[j - 1] > code) { E[j] = E[j - 1]; j--; }
            E[j] = code;
            int bw = c->w[lo * n + hi];
            agg += bw;                              /* Eq. 1 */
            if (bw == 50) x++;                      /* census */
            else if (bw == 25 || bw == 20) y++;
            else z++;
        }
        double s;
        if (c->selector == 0) s = agg;
        else if (c->selector == 1) s = c->sensitive ? oracle_eq2(x, y, z) : pres;
        else s = 0.0;
        int better = !u->found || s > u->score || (s == u->score && cmp_codes(E, u->E, m) < 0);
        if (better) {
            u->found = 1;
            u->score = s;
            for (int i = 0; i < k; i++) { u->S[i] = S[i]; u->pi[i] = perm[i]; }
            memcpy(u->E, E, sizeof(uint16_t) * m);
            u->agg = agg; u->x = x; u->y = y; u->z = z; u->pres = pres; u->eff = oracle_eq2(x, y, z);
        }
    } while (next_perm(rest, nr));
}

static void *deep_worker(void *arg) {
    dpool_t *p = (dpool_t *)arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int i = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (i >= p->nunits) break;
        deep_unit(p->c, p->subsets[i / p->c->k], i % p->c->k, &p->units[i]);
    }
    return NULL;
}

/* w: n*n weights; busy: bit d busy; pe: 2m pattern edges; selector as
 * oracle_allocate.  max_subsets bounds the work (error -2 above it).  Only the
 * subsets with lex index in [sub_lo, sub_hi) are scored (bounded samples and
 * shard tests; a negative bound = unrestricted). */
int oracle_allocate_deep(int n, const int32_t *w, uint64_t busy, int k, int m, const int32_t *pe,
                         int selector, int sensitive, int nthreads, int max_subsets, int sub_lo, int sub_hi,
                         oracle_result_deep *out) {
    memset(out, 0, sizeof(*out));
    if (n < 1 || n > 64 || k < 1 || k > 16 || m < 0 || m > 120) return -1;
    ctx_t c;
    c.n = n; c.k = k; c.m = m; c.selector = selector; c.sensitive = sensitive; c.w = w; c.pe = pe;
    c.nf = 0;
    for (int d = 0; d < n; d++)
        if (!((busy >> d) & 1ull)) c.F[c.nf++] = d;
    out->k = k;
    out->m = m;
    if (k > c.nf) { out->status = 1; return 0; }
    /* lex-ordered k-subsets of F */
    int cap = max_subsets > 0 ? max_subsets : 1;
    int (*subs)[16] = (int (*)[16])malloc(sizeof(int[16]) * (size_t)cap);
    int nsub = 0, idx[16];
    for (int i = 0; i < k; i++) idx[i] = i;
    for (;;) {
        if (nsub >= cap) { free(subs); return -2; }
        for (int i = 0; i < k; i++) subs[nsub][i] = c.F[idx[i]];
        nsub++;
        int i = k - 1;
        while (i >= 0 && idx[i] == c.nf - k + i) i--;
        if (i < 0) break;
        idx[i]++;
        for (int j = i + 1; j < k; j++) idx[j] = idx[j - 1] + 1;
    }
    int s_lo = sub_lo < 0 ? 0 : (sub_lo < nsub ? sub_lo : nsub);
    int s_hi = sub_hi < 0 ? nsub : (sub_hi < nsub ? sub_hi : nsub);
    if (s_hi < s_lo) s_hi = s_lo;
    memmove(subs, subs + s_lo, sizeof(int[16]) * (size_t)(s_hi - s_lo));
    nsub = s_hi - s_lo;
    dpool_t p;
    p.c = &c;
    p.subsets = subs;
    p.nsub = nsub;
    p.nunits = nsub * k;
    p.next = 0;
    p.units = (dunit_t *)calloc((size_t)p.nunits, sizeof(dunit_t));
    pthread_mutex_init(&p.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, deep_worker, &p);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&p.mu);
    dunit_t best;
    memset(&best, 0, sizeof(best));
    uint64_t raw = 0;
    for (int i = 0; i < p.nunits; i++) {            /* combine in (subset, pi[0]) order */
        dunit_t *u = &p.units[i];
        raw += u->raw;
        if (!u->found) continue;
        int same_set = best.found && memcmp(u->S, best.S, sizeof(int) * k) == 0;
        if (!best.found || u->score > best.score ||
            (u->score == best.score && same_set && cmp_codes(u->E, best.E, m) < 0))
            best = *u;
    }
    free(p.units);
    free(subs);
    out->raw = raw;
    out->status = best.found ? 0 : 1;
    if (!best.found) return 0;
    out->score = best.score;
    for (int i = 0; i < k; i++) {
        out->device_mask |= 1ull << best.S[i];
        out->mapping[i] = (int8_t)best.pi[i];
    }
    for (int i = 0; i < m; i++) { out->used[i][0] = best.E[i] >> 6; out->used[i][1] = best.E[i] & 63; }
    out->x = best.x; out->y = best.y; out->z = best.z;
    out->agg_bw = best.agg; out->preserved_bw = best.pres; out->pred_effbw = best.eff;
    return 0;
}
