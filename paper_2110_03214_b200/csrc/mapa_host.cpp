// mapa_host.cpp — host side of libmapa: topology encode (S1), pattern compile
// (S2), Eq. 2 rank tables, launch planning, key decode (S8) and the C-ABI.
// Nothing here enumerates or scores embeddings: that is esa.cu.  The decode
// recomputes the winner's census / scores from (S, mapping) only to report
// them and to self-check the key.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "internal.h"

#include <nvtx3/nvToolsExt.h>

using namespace mapa;

// One cached mapa_allocate sequence (H2D query, record zeroing, kernel, D2H
// record) as an instantiated CUDA graph, keyed by (pattern uid, selector /
// flags / path, free count, device): the kernel's parameters depend only on
// those; the busy mask itself is read from the pinned staging buffer when the
// graph runs.
struct GraphEntry {
    uint64_t key[3];
    cudaGraphExec_t exec;
    uint64_t tick;
};

// mapa_allocate_many: one cached graph per (patterns, selectors, flags, |F|, device)
struct ManyEntry {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec;
    uint64_t tick;
};

struct mapa_topology {
    std::string name;
    int n = 0;
    int width = 8;
    uint8_t cls[kMaxNDeep][kMaxNDeep];   // class code 0..3, diagonal 0xFF
    std::vector<std::vector<int>> sockets;
    uint64_t busy = 0;
    int dev = -1;                 // device of the stream / staging state below (set on first use)
    void *d_stage = nullptr;      // device: query (16 B) + record (32 / 64 B)
    void *h_stage = nullptr;      // pinned host mirror
    cudaStream_t cap = nullptr;   // private stream for graph capture (the caller's may be the legacy stream)
    std::vector<cudaStream_t> side;  // mapa_launch_queries' fork streams
    // mapa_launch_queries' small-query batch: device [counter (64 B) | order],
    // its pinned host staging, and the event guarding the staging's reuse
    void *d_mix = nullptr, *h_mix = nullptr;
    size_t mix_cap = 0;
    cudaEvent_t ev_mix = nullptr;
    // deep-path launch plans (suffix length, tuple table, terms, depth, grid)
    // keyed by (pattern uid, selector code, |F|, N, world): planning costs
    // far more host time than a small deep launch
    struct DeepPlanEntry { uint64_t key[3]; DeepTables tb; int sc, depth, stripe, grid; uint64_t tick; };
    std::vector<std::unique_ptr<DeepPlanEntry>> deep_plans;
    struct PairTab { int xs, dev; void *d; };
    std::vector<PairTab> pair_tabs;  // device images of the narrow kernels' pair tables, per (xs, device)
    std::vector<GraphEntry> graphs;
    std::vector<ManyEntry> many_graphs;
    void *d_many = nullptr, *h_many = nullptr;  // mapa_allocate_many staging: 128 B per query
    int many_cap = 0;
    uint64_t tick = 0;
};

struct mapa_pattern {
    int k = 0, m = 0;
    std::vector<std::pair<int, int>> edges;  // a < b, sorted
    uint16_t adj[kMaxKDeep];   // adjacency masks
    uint16_t back[kMaxKDeep];  // back[j] bit i: edge (i, j), i < j
    uint16_t src[kMaxKDeep];   // src[u] bit i: lex-leader f(i) < f(u)
    uint64_t aut = 1;          // |Aut(P)| (16! < 2^45)
    std::vector<uint16_t> lut;   // (m+1)^2
    double theta[14];          // Eq. 2 model of this pattern (Table 4 unless mapa_pattern_set_effbw_model)
    // device copies of the rank (+ bound) table for the deep kernel, one per
    // device, uploaded on first use and kept until the model changes (cached
    // graphs on any device may hold the pointer of theirs)
    std::vector<std::pair<int, void *>> d_luts;
    uint64_t uid = 0;          // unique per compiled pattern / model (graph cache key)
    // Eq. 3 set search (deep path, MAPA_F_PRUNE): the full-k pattern, and the
    // pattern's lex-smallest used-edge list over rank pairs (weight independent)
    mapa_pattern *clique = nullptr;
    bool have_ecode_min = false;
    uint64_t ecode_min[2] = {0, 0};
};

namespace {

// NVTX range over a C-ABI entry point (SURVEY §5 tracing; header-only NVTX v3:
// a no-op unless a profiler injects itself)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

thread_local std::string g_err;

mapa_status fail(mapa_status st, const std::string &msg) {
    g_err = msg;
    return st;
}

// ------------------------------------------------------------------ topology
// Link classes, Table 1.
const char *kClassNames[4] = {"nv2x2", "nv2x1", "nv1x1", "pcie"};

void topo_init(mapa_topology *t, const std::string &name, int n) {
    t->name = name;
    t->n = n;
    t->width = n <= 8 ? 8 : (n <= 16 ? 16 : (n <= 32 ? 32 : 64));
    for (int u = 0; u < kMaxNDeep; ++u)
        for (int v = 0; v < kMaxNDeep; ++v) t->cls[u][v] = (u == v) ? 0xFF : 3;  // PCIe fallback
}

void topo_link(mapa_topology *t, int a1, int b1, int c) {  // 1-based ids
    t->cls[a1 - 1][b1 - 1] = (uint8_t)c;
    t->cls[b1 - 1][a1 - 1] = (uint8_t)c;
}

// DGX-1 hybrid cube-mesh wiring, SPEC S:46 (classes fixed by P:261 and the
// §2.2 worked examples P:294).
const int kCubeDouble[8][2] = {{1, 4}, {1, 5}, {2, 3}, {2, 6}, {3, 4}, {5, 8}, {6, 7}, {7, 8}};
const int kCubeSingle[8][2] = {{1, 2}, {1, 3}, {2, 4}, {3, 7}, {4, 8}, {5, 6}, {5, 7}, {6, 8}};

bool build_builtin(const std::string &name, mapa_topology *t) {
    if (name == "dgx1v" || name == "dgx1p") {
        topo_init(t, name, 8);
        const bool p100 = name == "dgx1p";
        for (auto &e : kCubeDouble) topo_link(t, e[0], e[1], p100 ? 2 : 0);
        for (auto &e : kCubeSingle) topo_link(t, e[0], e[1], p100 ? 2 : 1);
        t->sockets = {{0, 1, 2, 3}, {4, 5, 6, 7}};
        return true;
    }
    if (name == "summit") {
        topo_init(t, name, 6);
        for (int s = 0; s < 2; ++s)
            for (int a = 1; a <= 3; ++a)
                for (int b = a + 1; b <= 3; ++b) topo_link(t, 3 * s + a, 3 * s + b, 0);
        t->sockets = {{0, 1, 2}, {3, 4, 5}};
        return true;
    }
    if (name == "torus2d16") {  // rows DoubleNVLink2, columns SingleNVLink2
        topo_init(t, name, 16);
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
                const int u = 4 * r + c + 1;
                topo_link(t, u, 4 * r + (c + 1) % 4 + 1, 0);
                topo_link(t, u, 4 * ((r + 1) % 4) + c + 1, 1);
            }
        t->sockets = {{0, 1, 2, 3, 4, 5, 6, 7}, {8, 9, 10, 11, 12, 13, 14, 15}};
        return true;
    }
    if (name == "cubemesh16") {
        topo_init(t, name, 16);
        for (int o = 0; o <= 8; o += 8) {
            for (auto &e : kCubeDouble) topo_link(t, e[0] + o, e[1] + o, 0);
            for (auto &e : kCubeSingle) topo_link(t, e[0] + o, e[1] + o, 1);
        }
        const int br[4][2] = {{1, 9}, {4, 12}, {5, 13}, {8, 16}};
        for (auto &e : br) topo_link(t, e[0], e[1], 1);
        t->sockets = {{0, 1, 2, 3, 4, 5, 6, 7}, {8, 9, 10, 11, 12, 13, 14, 15}};
        return true;
    }
    return false;
}

mapa_status parse_topology_text(const char *text, mapa_topology *t) {
    std::istringstream in(text);
    std::string line;
    int ln = 0, n = -1;
    std::string name = "topology";
    std::vector<std::vector<int>> sockets;
    struct L { int a, b, c, line; };
    std::vector<L> links;
    while (std::getline(in, line)) {
        ++ln;
        const size_t hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        std::istringstream ls(line);
        std::string f;
        if (!(ls >> f)) continue;
        if (f == "name") {
            if (!(ls >> name)) return fail(MAPA_E_PARSE, "line " + std::to_string(ln) + ": name: missing value");
        } else if (f == "devices") {
            if (!(ls >> n) || n < 1) return fail(MAPA_E_PARSE, "line " + std::to_string(ln) + ": devices: bad count");
            if (n > kMaxNDeep) return fail(MAPA_E_UNSUPPORTED, "line " + std::to_string(ln) + ": devices > 64 unsupported");
        } else if (f == "sockets") {
            std::string grp;
            while (ls >> grp) {
                std::vector<int> s;
                std::istringstream gs(grp);
                std::string id;
                while (std::getline(gs, id, ',')) {
                    char *end = nullptr;
                    const long v = std::strtol(id.c_str(), &end, 10);
                    if (id.empty() || *end) return fail(MAPA_E_PARSE, "line " + std::to_string(ln) + ": sockets: bad id '" + id + "'");
                    s.push_back((int)v - 1);
                }
                sockets.push_back(s);
            }
        } else if (f == "link") {
            int a, b;
            std::string c;
            if (!(ls >> a >> b >> c)) return fail(MAPA_E_PARSE, "line " + std::to_string(ln) + ": link: expected 'link a b class'");
            int code = -1;
            for (int i = 0; i < 4; ++i)
                if (c == kClassNames[i]) code = i;
            if (code < 0) return fail(MAPA_E_PARSE, "line " + std::to_string(ln) + ": link: unknown class '" + c + "'");
            links.push_back({a, b, code, ln});
        } else {
            return fail(MAPA_E_PARSE, "line " + std::to_string(ln) + ": unknown field '" + f + "'");
        }
    }
    if (n < 1) return fail(MAPA_E_PARSE, "missing 'devices'");
    topo_init(t, name, n);
    bool seen[kMaxNDeep][kMaxNDeep] = {};
    for (const L &l : links) {
        if (l.a == l.b) return fail(MAPA_E_PARSE, "line " + std::to_string(l.line) + ": link: self loop");
        if (l.a < 1 || l.b < 1 || l.a > n || l.b > n)
            return fail(MAPA_E_ID_RANGE, "line " + std::to_string(l.line) + ": link: id out of range");
        if (seen[l.a - 1][l.b - 1]) return fail(MAPA_E_PARSE, "line " + std::to_string(l.line) + ": link: duplicate edge");
        seen[l.a - 1][l.b - 1] = seen[l.b - 1][l.a - 1] = true;
        topo_link(t, l.a, l.b, l.c);
    }
    if (sockets.empty()) {
        std::vector<int> all;
        for (int i = 0; i < n; ++i) all.push_back(i);
        sockets.push_back(all);
    }
    std::vector<int> cover(n, 0);
    for (auto &s : sockets)
        for (int d : s) {
            if (d < 0 || d >= n) return fail(MAPA_E_ID_RANGE, "sockets: id out of range");
            cover[d]++;
        }
    for (int d = 0; d < n; ++d)
        if (cover[d] != 1) return fail(MAPA_E_PARSE, "sockets: groups must be disjoint and cover every device");
    t->sockets = sockets;
    return MAPA_OK;
}

void fill_devtopo(const mapa_topology *t, DevTopo &dt) {
    std::memset(&dt, 0, sizeof(dt));
    dt.n = t->n;
    dt.width = t->width;
    for (int v = 0; v < t->n; ++v)
        for (int u = 0; u < t->n; ++u)
            if (u != v) dt.cm[v][t->cls[u][v]] |= 1u << u;
}

int bw_of(const mapa_topology *t, int u, int v) { return kClassBw[t->cls[u][v]]; }

uint64_t nmask_of(int n) { return n >= 64 ? ~0ull : ((1ull << n) - 1ull); }

// ---------------------------------------------------------------- Eq. 2
// Predicted effective bandwidth, Eq. 2, Table 4.
const double kTheta[14] = {16.396, 4.536, 1.556, -20.694, -9.467, 7.615, -7.973,
                           12.733, -4.195, -8.413, 62.851, 27.418, -5.114, -46.973};

// The 14 features of Eq. 2 (the model is linear in theta).
void eq2_features(int xi, int yi, int zi, double *f) {
    const double x = xi, y = yi, z = zi;
    f[0] = x; f[1] = y; f[2] = z;
    f[3] = 1.0 / (x + 1.0); f[4] = 1.0 / (y + 1.0); f[5] = 1.0 / (z + 1.0);
    f[6] = x * y; f[7] = y * z; f[8] = z * x;
    f[9] = 1.0 / (x * y + 1.0); f[10] = 1.0 / (y * z + 1.0); f[11] = 1.0 / (z * x + 1.0);
    f[12] = x * y * z; f[13] = 1.0 / (x * y * z + 1.0);
}

double eq2_theta(const double *th, int xi, int yi, int zi) {
    const double x = xi, y = yi, z = zi;
    const double lin = th[0] * x + th[1] * y + th[2] * z;
    const double inv = th[3] / (x + 1.0) + th[4] / (y + 1.0) + th[5] / (z + 1.0);
    const double pair = th[6] * x * y + th[7] * y * z + th[8] * z * x;
    const double ipair = th[9] / (x * y + 1.0) + th[10] / (y * z + 1.0) + th[11] / (z * x + 1.0);
    const double trip = th[12] * x * y * z + th[13] / (x * y * z + 1.0);
    return lin + inv + pair + ipair + trip;
}

double eq2(int xi, int yi, int zi) { return eq2_theta(kTheta, xi, yi, zi); }

// Dense rank of Eq. 2 over the censuses with x+y+z = m (reading A9/A20: with
// Table 4 theta distinct censuses never tie and double order is exact; with a
// fitted theta the double order defines the rank).
std::vector<uint16_t> rank_table(int m, const double *th = kTheta) {
    std::vector<std::pair<double, int>> v;
    for (int x = 0; x <= m; ++x)
        for (int y = 0; x + y <= m; ++y) v.push_back({eq2_theta(th, x, y, m - x - y), x * (m + 1) + y});
    std::sort(v.begin(), v.end());
    std::vector<uint16_t> lut((size_t)(m + 1) * (m + 1), 0);
    int r = 0;
    for (size_t i = 0; i < v.size(); ++i) {
        if (i > 0 && v[i].first != v[i - 1].first) ++r;
        lut[v[i].second] = (uint16_t)r;
    }
    return lut;
}

// ---------------------------------------------------------------- patterns
uint64_t next_uid() {
    static std::atomic<uint64_t> c{1};
    return c.fetch_add(1);
}

// Does an automorphism sigma of P exist with sigma(j) = j for j < i and
// sigma(i) = u?  Backtracking over sigma(v), v = i+1..k-1, keeping adjacency
// AND non-adjacency with every assigned vertex (so a complete sigma is an
// automorphism) and equal degrees.
bool aut_extends(const mapa_pattern *p, int v, int *sig, uint32_t used) {
    const int k = p->k;
    if (v == k) return true;
    for (int c = 0; c < k; ++c) {
        if ((used >> c) & 1u) continue;
        if (__builtin_popcount(p->adj[c]) != __builtin_popcount(p->adj[v])) continue;
        bool ok = true;
        for (int w = 0; w < v && ok; ++w)
            ok = ((p->adj[v] >> w) & 1u) == ((p->adj[c] >> sig[w]) & 1u);
        if (!ok) continue;
        sig[v] = c;
        if (aut_extends(p, v + 1, sig, used | (1u << c))) return true;
    }
    return false;
}

mapa_status compile_pattern(int k, const std::vector<std::pair<int, int>> &raw, uint32_t flags,
                            mapa_pattern **out) {
    if (k < 1 || k > kMaxKDeep) return fail(MAPA_E_UNSUPPORTED, "pattern: need 1 <= k <= 16");
    mapa_pattern *p = new (std::nothrow) mapa_pattern();
    if (!p) return fail(MAPA_E_INVALID_ARG, "out of memory");
    p->k = k;
    std::memset(p->adj, 0, sizeof(p->adj));
    for (auto e : raw) {
        int a = e.first, b = e.second;
        if (a < 0 || b < 0 || a >= k || b >= k) { delete p; return fail(MAPA_E_INVALID_ARG, "pattern: vertex id out of range"); }
        if (a == b) { delete p; return fail(MAPA_E_INVALID_ARG, "pattern: self loop"); }
        if (a > b) std::swap(a, b);
        if ((p->adj[a] >> b) & 1u) { delete p; return fail(MAPA_E_INVALID_ARG, "pattern: duplicate edge"); }
        p->adj[a] |= (uint16_t)(1u << b);
        p->adj[b] |= (uint16_t)(1u << a);
        p->edges.push_back({a, b});
    }
    std::sort(p->edges.begin(), p->edges.end());
    p->m = (int)p->edges.size();
    if (k > 1 && !(flags & MAPA_F_ALLOW_DISCONNECTED)) {
        uint32_t vis = 1, frontier = 1;
        while (frontier) {
            uint32_t nxt = 0;
            for (int u = 0; u < k; ++u)
                if ((frontier >> u) & 1u) nxt |= p->adj[u];
            frontier = nxt & ~vis;
            vis |= nxt;
        }
        if (vis != (k >= 32 ? 0xFFFFFFFFu : ((1u << k) - 1u))) {
            delete p;
            return fail(MAPA_E_DISCONNECTED, "pattern: disconnected (k > 1)");
        }
    }
    for (int j = 0; j < k; ++j) p->back[j] = (uint16_t)(p->adj[j] & ((1u << j) - 1u));
    // Point-stabiliser chain of Aut(P): the orbit of i under the automorphisms
    // fixing 0..i-1.  Every u != i in it gets the lex-leader constraint
    // f(i) < f(u); this keeps exactly the lex-min mapping of every Aut-orbit
    // (DESIGN.md).  |Aut| = product of the orbit sizes (orbit-stabiliser).
    std::memset(p->src, 0, sizeof(p->src));
    p->aut = 1;
    int sig[kMaxKDeep];
    for (int i = 0; i < k; ++i) {
        uint64_t orb = 0;
        for (int u = i; u < k; ++u) {
            for (int j = 0; j < i; ++j) sig[j] = j;
            bool ok = __builtin_popcount(p->adj[u]) == __builtin_popcount(p->adj[i]);
            for (int w = 0; w < i && ok; ++w) ok = ((p->adj[i] >> w) & 1u) == ((p->adj[u] >> w) & 1u);
            if (!ok) continue;
            sig[i] = u;
            if (!aut_extends(p, i + 1, sig, ((1u << i) - 1u) | (1u << u))) continue;
            ++orb;
            if (u != i) p->src[u] |= (uint16_t)(1u << i);
        }
        p->aut *= orb;
    }
    std::memcpy(p->theta, kTheta, sizeof(kTheta));
    p->lut = rank_table(p->m);
    p->uid = next_uid();
    *out = p;
    return MAPA_OK;
}

void fill_devpattern(const mapa_pattern *p, bool raw, uint16_t lut_off, DevPattern &dp) {
    std::memset(&dp, 0, sizeof(dp));
    dp.k = (uint8_t)p->k;
    dp.m = (uint8_t)p->m;
    dp.eb = (uint8_t)(p->k * (p->k - 1) / 2);
    dp.clique = p->m == dp.eb;
    for (int j = 0; j < p->k; ++j) {
        for (int u = j + 1; u < p->k; ++u) {
            if ((p->adj[j] >> u) & 1u) dp.fwd_back[j] |= (uint8_t)(1u << u);
            if (!raw && ((p->src[u] >> j) & 1)) dp.fwd_src[j] |= (uint8_t)(1u << u);
        }
        dp.dback[j] = (uint8_t)__builtin_popcount(p->back[j]);
    }
    for (int e = 0; e < p->m; ++e) dp.edge[e] = (uint8_t)(p->edges[e].first | (p->edges[e].second << 4));
    dp.lut_off = lut_off;
    dp.aut = (uint16_t)p->aut;
}

// narrow path: k <= 8 and the packed 63-bit key fits
bool key_fits(const mapa_topology *t, const mapa_pattern *p) {
    return t->n <= kMaxN && p->k <= kMaxK && 15 + t->width + p->k * (p->k - 1) / 2 <= 63;
}

uint64_t perm_count(int n, int d) {
    uint64_t r = 1;
    for (int j = 0; j < d; ++j) r *= (uint64_t)(n - j);
    return r;
}

// Row stride of the device Eq. 2 table (index x*xs + y, x, y <= m): the
// smallest xs >= m+1 such that lanes whose census differs by a small
// (dx, dy) rarely hit the same shared-memory bank (32 banks of 4 B):
// minimises #{(dx, dy) != 0, |dx|,|dy| <= 5 : 32 | xs*dx + dy}.
int pick_xs(int m) {
    // Row stride of the Eq. 2 table index x*xs + y.  The lanes of a warp read
    // entries whose censuses differ by small (dx, dy) with few 12-links
    // (|dx + dy| small); a pair conflicts on a shared-memory bank when
    // xs*dx + dy == 0 (mod 32).  Score each xs by the conflicting pairs,
    // weighted by how likely such a census difference is, and keep the
    // cheapest (ties: the smallest table).
    int best = m + 1;
    double bestc = 1e30;
    for (int xs = m + 1; xs <= std::max(m + 1, 40); ++xs) {
        double cost = 0.0;
        for (int dx = -6; dx <= 6; ++dx)
            for (int dy = -6; dy <= 6; ++dy)
                if ((dx || dy) && ((xs * dx + dy) % 32 + 32) % 32 == 0)
                    cost += std::exp(-0.5 * (std::abs(dx) + std::abs(dy) + std::abs(dx + dy)));
        if (cost < bestc - 1e-12) { bestc = cost; best = xs; }
    }
    return best;
}

mapa_status cuda_fail(int err, const char *what) {
    return fail(MAPA_E_CUDA, std::string(what) + ": " + cuda_error_string(err));
}

// Device image of the ten pair tables for (topology, Eq. 2 row stride xs) on
// the current device, built once (the single-query kernels copy it into
// shared memory instead of recomputing it in every CTA).  Null on failure:
// the kernel then builds the tables itself.
const int4 *pair_tables(const mapa_topology *tc, int xs, void *stream) {
    mapa_topology *t = const_cast<mapa_topology *>(tc);  // a cache of immutable data
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    for (auto &pt : t->pair_tabs)
        if (pt.xs == xs && pt.dev == dev) return (const int4 *)pt.d;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing((cudaStream_t)stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        return nullptr;  // never allocate inside a capture (mapa_allocate warms the cache first)
    DevTopo dt;
    fill_devtopo(t, dt);
    std::vector<int> img((size_t)kPairTables * kMaxN * kMaxN);
    for (int i = 0; i < kMaxN * kMaxN; ++i) {
        int e[kPairTables];
        pair_table_entry(dt, i, xs, e);
        for (int k = 0; k < kPairTables; ++k) img[(size_t)k * kMaxN * kMaxN + i] = e[k];
    }
    void *d = nullptr;
    if (cudaMalloc(&d, img.size() * sizeof(int)) != cudaSuccess) return nullptr;
    // pageable copy: make sure the DMA is complete before any stream reads it
    if (cudaMemcpy(d, img.data(), img.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    t->pair_tabs.push_back({xs, dev, d});
    return (const int4 *)d;
}

// Can the single-query Eq. 1 / Eq. 3 scans run on 16-bit lanes (SelT::lin16,
// esa_kernels.cuh)?  Their table entries are 32 (t2 + ishift) with t2 <= 50 (k-2)
// (the vertex k-2 has at most k-2 placed neighbours) for Eq. 1, and t2 =
// sum_U w(u, v) - inc_F(v), ishift = max_{v in F} inc_F(v) for Eq. 3, so
// t2 + ishift <= 50 (k-2) + spread, spread = max - min of inc_F over F
// (unknown F: spread <= max_v inc over all devices); entries must stay <= 31135.
// `bound`: kLin16Max (prune-mode kernels) or kLin16StatMax (the others)
bool lin16_fits(const mapa_topology *t, const mapa_pattern *p, int selcode, uint64_t busy_hint, int bound) {
    if (t->width < 16 || p->k < 3 || (selcode != SEL_GREEDY && selcode != SEL_INSENS)) return false;
    int spread = 0;
    if (selcode == SEL_INSENS) {
        const uint64_t all = nmask_of(t->n);
        const uint64_t F = busy_hint == ~0ull ? all : (~busy_hint & all);
        int lo = 1 << 30, hi = 0;
        for (int v = 0; v < t->n; ++v) {
            if (!((F >> v) & 1u)) continue;
            int inc = 0;
            for (int u = 0; u < t->n; ++u)
                if (u != v && ((F >> u) & 1u)) inc += bw_of(t, u, v);
            lo = std::min(lo, inc);
            hi = std::max(hi, inc);
        }
        spread = busy_hint == ~0ull ? hi : hi - (lo > hi ? hi : lo);
    }
    return 32 * (50 * (p->k - 2) + spread) <= bound;
}

struct Plan {
    int depth, chunk, grid;
    uint64_t nlocal;
};

bool has_constraints(const DevPattern &dp) {
    for (int j = 0; j < 8; ++j)
        if (dp.fwd_src[j]) return true;
    return false;
}

int multi_has_constraints(const MultiTables &tb) {
    for (int i = 0; i < tb.npats; ++i)
        if (has_constraints(tb.pat[i])) return 1;
    return 0;
}

Plan plan_single(const mapa_topology *t, const mapa_pattern *p, int sensk, int nF, int world) {
    Plan pl{};
    const int W = t->width, G = 32 / W, k = p->k;
    int sm = device_sm_count();
    if (sm <= 0) sm = 148;
    const int occ = max_blocks_per_sm_single(W, k, sensk, pick_xs(p->m));
    const uint64_t resident_warps = (uint64_t)sm * occ * 8;
    // Items = prefixes of depth D; guided self-scheduling balances ~8 items
    // per resident W-lane group, and D = k-3 (one inner3 call per item) is
    // reached whenever that gives enough items.
    // Going deeper than k-3 trades the lane-parallel inner3 path for more,
    // smaller items; do it only when a rank would have fewer items than
    // resident groups at k-3 (a sharded launch has 1/world of the items, so
    // the balance target alone would push every multi-rank launch deeper:
    // C4 at world 8 measured 59 us per kernel at k-2 vs ~28 us at k-3).
    const uint64_t target = 8ull * resident_warps * G * (uint64_t)world;
    int dmax = k <= 1 ? 0 : std::max(1, std::min(k - 2, 4));
    int d = k <= 1 ? 0 : 1;
    while (d < dmax && perm_count(nF, d) < target) {
        if (d >= k - 3 && perm_count(nF, d) >= resident_warps * G * (uint64_t)world) break;
        ++d;
    }
    pl.depth = d;
    const uint64_t items = nF >= k ? perm_count(nF, d) : 0;
    pl.nlocal = items;
    // Sharding: `chunk` is the stripe length; rank r owns stripes r, r+world, ...
    // (64 stripes per rank keep canonical-mode work balanced).  Inside a rank
    // the kernel hands out chunks by guided self-scheduling.
    uint64_t stripe = world == 1 ? std::max<uint64_t>(1, items)
                                 : std::max<uint64_t>(1, (items + 64ull * world - 1) / (64ull * world));
    pl.chunk = (int)std::min<uint64_t>(stripe, 1u << 30);
    const uint64_t local = (items + world - 1) / world;
    const uint64_t blocks = std::max<uint64_t>(1, (local + 8 * G - 1) / (8 * G));  // >= 1 item per group
    pl.grid = (int)std::min<uint64_t>(blocks, (uint64_t)sm * occ);
    return pl;
}

// ------------------------------------------------------------------ deep path
// Plan of one deep launch (esa_deep.cu): suffix length L, its tuple table, the
// decoded prefix depth D, the stripe and the grid.
struct DeepPlan {
    int sc, depth, stripe, grid;
    uint64_t items;
};

// Suffix-internal scored pairs for suffix length L: Eq. 3 every pair, Eq. 1 /
// Eq. 2 the pattern edges, Baseline none.
int suffix_pairs(const mapa_pattern *p, int L, int base, uint8_t (*es)[2]) {
    const int T = p->k - L;
    int n = 0;
    for (int a = 0; a < L; ++a)
        for (int b = a + 1; b < L; ++b) {
            const bool e = base == SEL_INSENS || (base != SEL_BASE && ((p->adj[T + a] >> (T + b)) & 1u));
            if (e) { es[n][0] = (uint8_t)a; es[n][1] = (uint8_t)b; ++n; }
        }
    return n;
}

// Terms of a tuple's score for suffix length L (DeepTables::term): Eq. 1 / 2
// the partial of every suffix vertex with a scored prefix neighbour plus the
// suffix-internal pattern edges; Eq. 3 with L >= 2 the C(L,2) pairs alone
// (pair folding, scale L-1), with L = 1 the single partial; Baseline none.
int suffix_terms(const mapa_pattern *p, int L, int base, uint8_t (*term)[3], int *nes, int *scale) {
    const int T = p->k - L;
    uint8_t es[8][2];
    *nes = suffix_pairs(p, L, base, es);
    const bool fold = base == SEL_INSENS && L >= 2;
    *scale = fold ? L - 1 : 1;
    int n = 0;
    uint8_t tmp[16][3];
    if (!fold && base != SEL_BASE)
        for (int l = 0; l < L; ++l)
            if (base == SEL_INSENS || (p->back[T + l] & ((1u << T) - 1u))) { tmp[n][0] = 0; tmp[n][1] = (uint8_t)l; tmp[n][2] = 0; ++n; }
    for (int e = 0; e < *nes; ++e) { tmp[n][0] = 1; tmp[n][1] = es[e][0]; tmp[n][2] = es[e][1]; ++n; }
    if (term)
        for (int i = 0; i < n && i < kDeepMaxTerms; ++i) std::memcpy(term[i], tmp[i], 3);
    return n;
}

// Valid L-tuples of distinct indices into r sorted devices (lex order); the
// suffix-internal lex-leader constraints f(T+a) < f(T+b) become i_a < i_b.
// Entry byte l = i_l.  Returns the count, or -1 above cap.
int build_tuples(const mapa_pattern *p, int L, int r, bool canon, uint32_t *out, int cap) {
    const int T = p->k - L;
    int n = 0, idx[4] = {0, 0, 0, 0};
    int total = 1;
    for (int l = 0; l < L; ++l) total *= r;
    for (int t = 0; t < total; ++t) {
        int x = t;
        for (int l = L - 1; l >= 0; --l) { idx[l] = x % r; x /= r; }
        bool ok = true;
        for (int a = 0; a < L && ok; ++a)
            for (int b = a + 1; b < L && ok; ++b) {
                if (idx[a] == idx[b]) ok = false;
                else if (canon && ((p->src[T + b] >> (T + a)) & 1u) && !(idx[a] < idx[b])) ok = false;
            }
        if (!ok) continue;
        if (n >= cap) return -1;
        uint32_t w = 0;
        for (int l = 0; l < L; ++l) w |= (uint32_t)idx[l] << (8 * l);
        if (out) out[n] = w;
        ++n;
    }
    if (out) {
        // order by the largest index, so that the tuples using only the first
        // r' devices form a prefix of the table (a node whose common lower
        // bound leaves r' devices scans tcount[r'] entries)
        // (a stable counting sort on the largest index: O(n + r))
        std::vector<uint32_t> tmp(out, out + n);
        std::vector<int> start(r + 1, 0);
        auto mx = [L](uint32_t w) {
            uint32_t m = 0;
            for (int l = 0; l < L; ++l) m = std::max(m, (w >> (8 * l)) & 0xFFu);
            return m;
        };
        for (int i = 0; i < n; ++i) ++start[mx(tmp[i]) + 1];
        for (int v = 0; v < r; ++v) start[v + 1] += start[v];
        for (int i = 0; i < n; ++i) out[start[mx(tmp[i])]++] = tmp[i];
    }
    return n;
}

// Eq. 2 branch and bound is built when the per-depth bound tables fit:
// (k + 1) tables of (m + 1)^2 u16 (<= 34 KB of shared memory)
bool sens_prunable(const mapa_pattern *p) { return (p->k + 1) * (p->m + 1) * (p->m + 1) <= kSensBoundMax; }

mapa_status plan_deep(const mapa_topology *t, const mapa_pattern *p, int selector, int sens, uint32_t flags,
                      int nF, int world, DeepTables *tb, DeepPlan *pl) {
    const int k = p->k;
    const bool canon = !(flags & MAPA_F_RAW) && p->aut > 1;
    const int base = sel_code(selector, sens);
    std::memset(tb, 0, sizeof(*tb));
    for (int v = 0; v < t->n; ++v)
        for (int u = 0; u < t->n; ++u)
            if (u != v && t->cls[u][v] < 3) tb->cm[v][t->cls[u][v]] |= 1ull << u;
    tb->n = t->n;
    tb->k = k;
    tb->m = p->m;
    tb->xsd = p->m + 1;
    tb->eb = k * (k - 1) / 2;
    tb->clique = p->m == tb->eb;
    for (int u = 0; u < k; ++u) {
        tb->back[u] = p->back[u];
        tb->src[u] = canon ? p->src[u] : 0;
    }
    for (int e = 0; e < p->m; ++e) tb->edge[e] = (uint8_t)(p->edges[e].first | (p->edges[e].second << 4));
    for (int u = 0; u < k; ++u) tb->adj[u] = p->adj[u];
    for (int d = 0; d <= k; ++d) {
        int c = 0;
        for (auto &e : p->edges) c += (e.first >= d && e.second >= d);
        tb->c2[d] = (uint8_t)c;
    }
    // suffix length L: smallest modelled cost per leaf (node overhead + rounds of 32 lanes)
    double best = 1e30;
    int bestL = 0;
    bool bestLanes2 = false;
    // parallelism: the warps can only split the prefix levels 0..k-L-1
    // (decoded items); with fewer prefixes than ~4 per resident warp of every
    // rank, most warps idle
    auto par = [&](int L) {
        const uint64_t want = 4ull * 148 * 3 * 8 * (uint64_t)world;
        const uint64_t avail = perm_count(nF, std::min(k - L, 6));
        return avail < want ? (double)want / (double)std::max<uint64_t>(1, avail) : 1.0;
    };
    for (int L = 1; L <= std::min(k, 4); ++L) {
        const int r = nF - k + L;
        if (r < L || r > kMaxNDeep) continue;
        if (L == 2) {
            // lanes2: vertex T loops over r devices, T+1 on the lanes (one or two
            // rounds of 32); no tuple table, so r is not capped at 16
            const bool dep = canon && ((p->src[k - 1] >> (k - 2)) & 1u);
            const double leaves = dep ? 0.5 * r * (r - 1) : (double)r * (r - 1);
            const double node = 40.0 + 24.0 + 6.0 * k + 10.0;
            const double per_i = ((r + 31) / 32) * (base == SEL_SENS ? 10.0 : 8.0) + 4.0;
            const double cost = (node + per_i * r) / std::max(1.0, leaves) * par(L);
            if (cost < best * 0.98) { best = cost; bestL = L; bestLanes2 = true; }
        }
        if (L >= 2 && r > 16) continue;
        const int nt = build_tuples(p, L, r, canon, nullptr, kMaxTup);
        if (nt <= 0) continue;
        int nes, scale;
        const int nterm = suffix_terms(p, L, base, nullptr, &nes, &scale);
        if (nterm > kDeepMaxTerms) continue;
        const int NT = nterm <= 2 ? 2 : (nterm <= 4 ? 4 : 6);
        const double node = 40.0 + 12.0 * L + (nes ? 6.0 * ((r * 16 + 31) / 32) : 0.0) + 6.0 * k;
        const double round = 12.0 + 3.0 * NT;
        const double cost = (node + round * ((nt + 31) / 32)) / nt * par(L);
        if (cost < best * 0.98) { best = cost; bestL = L; bestLanes2 = false; }
    }
    if (!bestL) return fail(MAPA_E_UNSUPPORTED, "deep path: no feasible suffix length");
    const int L = bestL, T = k - L, r = nF - T;
    tb->L = L;
    tb->T = T;
    tb->r = r;
    if (bestLanes2) {
        tb->lanes2 = 1;
        tb->l2e = base == SEL_INSENS || ((base == SEL_GREEDY || base == SEL_SENS) && ((p->adj[T] >> (T + 1)) & 1u));
        tb->l2dep = canon && ((p->src[T + 1] >> T) & 1u);
        tb->ntup = 0;
        tb->nterm = 2;  // the NT = 2 instantiation (no tuple terms are read)
        tb->nes = 0;
        tb->scale = 1;
    } else {
        tb->ntup = build_tuples(p, L, r, canon, tb->tup, kMaxTup);
        tb->nterm = suffix_terms(p, L, base, tb->term, &tb->nes, &tb->scale);
    }
    // prefix sources common to every suffix vertex: their max is a lower bound
    // for the whole suffix, applied by compacting the node's device list; the
    // remaining per-vertex bounds are checked per tuple (pcon)
    const uint32_t pmask = (1u << T) - 1u;
    uint32_t common = canon ? pmask : 0u;
    for (int l = 0; l < L; ++l) common &= p->src[T + l];
    tb->pcommon = (int32_t)common;
    tb->pcon = 0;
    if (canon)
        for (int l = 0; l < L; ++l)
            if (p->src[T + l] & pmask & ~common) tb->pcon = 1;
    {   // tcount[r'] = #tuples with largest index < r' (histogram + prefix sum)
        int hist[kMaxNDeep + 1] = {0};
        for (int i = 0; i < tb->ntup; ++i) {
            uint32_t m = 0;
            for (int l = 0; l < L; ++l) m = std::max(m, (tb->tup[i] >> (8 * l)) & 0xFFu);
            ++hist[m + 1 <= (uint32_t)kMaxNDeep ? m + 1 : kMaxNDeep];
        }
        int c = 0;
        for (int rr = 0; rr <= kMaxNDeep; ++rr) {
            c += hist[rr];
            tb->tcount[rr] = c;
        }
    }
    // branch and bound (MAPA_F_PRUNE): Greedy only.  (An Eq. 3 variant with
    // the bound (k-1) maxw[v] - inc_F(v) per later vertex was exact but pruned
    // nothing on cubemesh16 and cost 20-40 %: not dispatched.)
    const bool prune = (flags & MAPA_F_PRUNE) && (base == SEL_GREEDY || (base == SEL_SENS && sens_prunable(p)));
    pl->sc = base | (canon ? 4 : 0) | (prune ? 8 : 0);
    // decoded prefix depth: enough items for ~8 per resident warp (x world)
    int sm = device_sm_count();
    if (sm <= 0) sm = 148;
    // rank (+ bound) tables and the tuple table behind DeepShared
    const int lutb = (base == SEL_SENS ? 2 * tb->xsd * tb->xsd * (1 + (prune ? k + 1 : 0)) : 0) + 16 + 16 * tb->ntup;
    const int occ = max_blocks_per_sm_deep(t->n, tb->nterm, pl->sc, lutb);
    const uint64_t warps = (uint64_t)sm * occ * 8;
    const uint64_t target = 8ull * warps * (uint64_t)world;
    // RAW items are uniform: stop at ~8 per warp.  Canonical items are not
    // (the lex-leader bounds make prefixes with small devices first far
    // heavier, and they are contiguous in item order), so go as deep as the
    // 2^26-item budget allows: the heaviest item is then a small fraction of
    // a warp's share and guided self-scheduling balances the rest.
    int d = 0;
    while (d < std::min(T, 6) && (canon || perm_count(nF, d) < target) && perm_count(nF, d + 1) < (1ull << 26)) ++d;
    pl->depth = d;
    pl->items = perm_count(nF, d);
    const uint64_t stripe = world == 1 ? std::max<uint64_t>(1, pl->items)
                                       : std::max<uint64_t>(1, (pl->items + 64ull * world - 1) / (64ull * world));
    pl->stripe = (int)std::min<uint64_t>(stripe, 1u << 30);
    const uint64_t local = (pl->items + world - 1) / world;
    pl->grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((local + 7) / 8, (uint64_t)sm * occ));
    return MAPA_OK;
}

// Rank table followed, for Eq. 2 branch and bound, by one bound table per
// number of placed vertices nd: ub[nd][x*(m+1) + y] = the largest rank of a
// final census (x+a, y+b, .) with a + b <= c_nd, c_nd = the pattern edges not
// inside {0..nd-1} (exact: the remaining edges can only add to x, y or z).
std::vector<uint16_t> rank_and_bounds(const mapa_pattern *p) {
    std::vector<uint16_t> v(p->lut);
    if (!sens_prunable(p)) return v;
    const int m = p->m, xs = m + 1, k = p->k;
    for (int nd = 0; nd <= k; ++nd) {
        int inside = 0;
        for (auto &e : p->edges) inside += (e.first < nd && e.second < nd);
        const int c = m - inside;
        for (int x = 0; x < xs; ++x)
            for (int y = 0; y < xs; ++y) {
                int best = 0;
                if (x + y <= m)
                    for (int a2 = 0; a2 <= c && x + a2 <= m; ++a2)
                        for (int b2 = 0; a2 + b2 <= c && x + a2 + y + b2 <= m; ++b2)
                            best = std::max(best, (int)p->lut[(x + a2) * xs + (y + b2)]);
                v.push_back((uint16_t)best);
            }
    }
    return v;
}

mapa_status upload_lut(const mapa_pattern *pc, const uint16_t **out) {
    mapa_pattern *p = const_cast<mapa_pattern *>(pc);  // the device copy caches the immutable table
    int dev = 0, err;
    if ((err = (int)cudaGetDevice(&dev))) return cuda_fail(err, "cudaGetDevice");
    for (auto &e : p->d_luts)
        if (e.first == dev) {
            *out = (const uint16_t *)e.second;
            return MAPA_OK;
        }
    const std::vector<uint16_t> img = rank_and_bounds(p);
    const size_t bytes = img.size() * sizeof(uint16_t);
    void *d = nullptr;
    if ((err = (int)cudaMalloc(&d, bytes))) return cuda_fail(err, "cudaMalloc (rank table)");
    // a pageable copy may still be in flight when cudaMemcpy returns: finish it
    // before any stream (non-blocking ones included) can read the table
    if ((err = (int)cudaMemcpy(d, img.data(), bytes, cudaMemcpyHostToDevice)) ||
        (err = (int)cudaStreamSynchronize(cudaStreamLegacy))) {
        cudaFree(d);
        return cuda_fail(err, "H2D rank table");
    }
    p->d_luts.push_back({dev, d});
    *out = (const uint16_t *)d;
    return MAPA_OK;
}

void free_luts(mapa_pattern *p) {
    for (auto &e : p->d_luts) cudaFree(e.second);
    p->d_luts.clear();
}

// The topology's staging buffers, capture / side streams and cached graphs
// belong to the device current at their first use: mapa_allocate and
// mapa_launch_queries refuse a handle used from another device.
mapa_status bind_device(mapa_topology *t) {
    int dev = 0, err;
    if ((err = (int)cudaGetDevice(&dev))) return cuda_fail(err, "cudaGetDevice");
    if (t->dev < 0) t->dev = dev;
    if (t->dev != dev)
        return fail(MAPA_E_INVALID_ARG, "topology handle is bound to device " + std::to_string(t->dev) +
                                            " (current device " + std::to_string(dev) + "): use one handle per device");
    return MAPA_OK;
}

// Lex-first bijection pi: V(P) -> S (pattern-vertex order, devices ascending)
// with pi(E(P)) = E: keep adjacency and non-adjacency with every placed vertex
// and equal degrees; the first complete map is the lex-first one.
bool first_mapping(const mapa_pattern *p, const std::vector<int> &ds, const uint64_t *eadj, int v, int *pi,
                   uint64_t used) {
    const int k = p->k;
    if (v == k) return true;
    for (int c : ds) {
        if ((used >> c) & 1u) continue;
        if (__builtin_popcountll(eadj[c]) != __builtin_popcount(p->adj[v])) continue;
        bool ok = true;
        for (int w = 0; w < v && ok; ++w) ok = (((p->adj[v] >> w) & 1u) != 0) == (((eadj[c] >> pi[w]) & 1u) != 0);
        if (!ok) continue;
        pi[v] = c;
        if (first_mapping(p, ds, eadj, v + 1, pi, used | (1ull << c))) return true;
    }
    return false;
}

// Decision from (S, E) (both paths): lex-first mapping, census, Eq. 1/2/3, and
// the self-check of the key's score.
mapa_status fill_decision(const mapa_topology *t, const mapa_pattern *p, uint64_t F, uint64_t S,
                          std::vector<std::pair<int, int>> E, int selector, int sens, uint32_t score,
                          mapa_decision &d) {
    const int k = p->k;
    if (__builtin_popcountll(S) != k || (S & ~F)) return fail(MAPA_E_INTERNAL, "decoded device set inconsistent");
    if ((int)E.size() != p->m) return fail(MAPA_E_INTERNAL, "decoded edge set has wrong size");
    std::sort(E.begin(), E.end());
    std::vector<int> ds;
    for (int dv = 0; dv < t->n; ++dv)
        if ((S >> dv) & 1u) ds.push_back(dv);
    uint64_t eadj[kMaxNDeep] = {0};
    for (auto &e : E) { eadj[e.first] |= 1ull << e.second; eadj[e.second] |= 1ull << e.first; }
    int pi[kMaxKDeep];
    if (!first_mapping(p, ds, eadj, 0, pi, 0ull))
        return fail(MAPA_E_INTERNAL, "no mapping of the decoded set yields the decoded edges");
    int agg = 0, x = 0, y = 0, z = 0;
    for (auto &e : E) {
        const int c = t->cls[e.first][e.second];
        agg += kClassBw[c];
        if (c == 0) ++x;
        else if (c == 3) ++z;
        else ++y;
    }
    int pres = 0;
    for (int u = 0; u < t->n; ++u)
        for (int v = u + 1; v < t->n; ++v)
            if (((F >> u) & (F >> v) & 1u) && !((S >> u) & 1u) && !((S >> v) & 1u)) pres += bw_of(t, u, v);
    uint32_t expect = 0;
    if (selector == MAPA_SEL_GREEDY) expect = (uint32_t)agg;
    else if (selector == MAPA_SEL_PRESERVE) expect = sens ? p->lut[x * (p->m + 1) + y] : (uint32_t)pres;
    if (expect != score) return fail(MAPA_E_INTERNAL, "key score does not match the decoded match");
    d.status = MAPA_OK;
    d.device_mask = S;
    for (int i = 0; i < k; ++i) d.mapping[i] = (int8_t)pi[i];
    for (size_t i = 0; i < E.size(); ++i) { d.used[i][0] = E[i].first; d.used[i][1] = E[i].second; }
    d.x = x; d.y = y; d.z = z;
    d.agg_bw = agg;
    d.preserved_bw = pres;
    d.score = (int32_t)score;
    d.pred_effbw = eq2_theta(p->theta, x, y, z);
    return MAPA_OK;
}

mapa_status decode_wide(const mapa_topology *t, const mapa_pattern *p, uint64_t busy, int selector, int sens,
                        uint32_t flags, const mapa_wide_record *rec, mapa_decision *out) {
    mapa_decision d;
    std::memset(&d, 0, sizeof(d));
    d.k = p->k;
    d.m = p->m;
    d.key = rec->score;
    d.ecode[0] = rec->ecode_hi;
    d.ecode[1] = rec->ecode_lo;
    d.leaves_scored = rec->leaves;
    const uint64_t F = ~busy & nmask_of(t->n);
    if ((flags & MAPA_F_PRUNE) &&
        (selector == MAPA_SEL_GREEDY || (selector == MAPA_SEL_PRESERVE && sens && sens_prunable(p)))) {
        // the pruned kernel scores a subset; the totals are the closed forms
        uint64_t perm = 1;
        const int nf = __builtin_popcountll(F);
        for (int i = 0; i < p->k; ++i) perm *= (uint64_t)std::max(0, nf - i);
        d.raw_embeddings = perm;
        d.distinct_matches = perm / p->aut;
    } else if (flags & MAPA_F_RAW) {
        d.raw_embeddings = rec->leaves;
        d.distinct_matches = rec->leaves / p->aut;
    } else {
        d.distinct_matches = rec->leaves;
        d.raw_embeddings = rec->leaves * p->aut;
    }
    if (rec->status != 0)
        return fail(MAPA_E_INVALID_ARG, rec->status == 2 ? "device refused the query: static shared tables misplaced"
                                                          : "device reported a bad query (busy_hint != d_query->busy?)");
    if (rec->set == 0) {
        d.status = MAPA_NO_CAPACITY;
        *out = d;
        return MAPA_NO_CAPACITY;
    }
    const int k = p->k, eb = k * (k - 1) / 2;
    if (rec->score > 0xFFFFFFFFull) return fail(MAPA_E_INTERNAL, "score out of range");
    const uint32_t score = (uint32_t)rec->score;
    uint64_t S = 0;
    for (int dv = 0; dv < 64; ++dv)
        if ((rec->set >> (63 - dv)) & 1u) S |= 1ull << dv;
    std::vector<int> ds;
    for (int dv = 0; dv < 64; ++dv)
        if ((S >> dv) & 1u) ds.push_back(dv);
    if ((int)ds.size() != k) return fail(MAPA_E_INTERNAL, "decoded device set has wrong size");
    std::vector<std::pair<int, int>> E;
    int pidx = 0;
    for (int a = 0; a < k; ++a)
        for (int b = a + 1; b < k; ++b, ++pidx) {
            const int q = eb - 1 - pidx;
            const uint64_t bit = q >= 64 ? (rec->ecode_hi >> (q - 64)) & 1u : (rec->ecode_lo >> q) & 1u;
            if (bit) E.push_back({ds[a], ds[b]});
        }
    mapa_status st = fill_decision(t, p, F, S, E, selector, sens, score, d);
    if (st != MAPA_OK) return st;
    *out = d;
    return MAPA_OK;
}

mapa_status decode_record(const mapa_topology *t, const mapa_pattern *p, uint64_t busy, int selector,
                          int sens, uint32_t flags, const mapa_record *rec, mapa_decision *out) {
    mapa_decision d;
    std::memset(&d, 0, sizeof(d));
    d.k = p->k;
    d.m = p->m;
    d.key = rec->key;
    d.leaves_scored = rec->leaves;
    const bool raw = (flags & MAPA_F_RAW) != 0;
    const uint64_t F = ~busy & nmask_of(t->n);
    if ((flags & MAPA_F_PRUNE) && p->k >= 4) {
        // the pruned kernel scores a subset; the totals are the closed forms
        uint64_t perm = 1;
        const int nf = __builtin_popcountll(F);
        for (int i = 0; i < p->k; ++i) perm *= (uint64_t)std::max(0, nf - i);
        d.raw_embeddings = perm;
        d.distinct_matches = perm / (uint64_t)p->aut;
    } else if (raw) {
        d.raw_embeddings = rec->leaves;
        d.distinct_matches = rec->leaves / (uint64_t)p->aut;
    } else {
        d.distinct_matches = rec->leaves;
        d.raw_embeddings = rec->leaves * (uint64_t)p->aut;
    }
    if (rec->status != 0)
        return fail(MAPA_E_INVALID_ARG, rec->status == 2 ? "device refused the query: static shared tables misplaced"
                                                          : "device reported a bad query");
    if (rec->key == 0) {
        d.status = MAPA_NO_CAPACITY;
        *out = d;
        return MAPA_NO_CAPACITY;
    }
    const int W = t->width, eb = p->k * (p->k - 1) / 2, k = p->k;
    const uint64_t key = rec->key;
    const uint32_t score = (uint32_t)(key >> (W + eb));
    const uint32_t sb = (uint32_t)((key >> eb) & (W >= 32 ? 0xFFFFFFFFull : ((1ull << W) - 1)));
    const uint32_t ecode = (uint32_t)(key & ((1ull << eb) - 1));
    uint32_t S = 0;
    for (int dv = 0; dv < W; ++dv)
        if ((sb >> (W - 1 - dv)) & 1u) S |= 1u << dv;
    std::vector<int> ds;
    for (int dv = 0; dv < t->n; ++dv)
        if ((S >> dv) & 1u) ds.push_back(dv);
    if ((int)ds.size() != k) return fail(MAPA_E_INTERNAL, "decoded device set inconsistent");
    // used-edge set from the edge code (pair p in lex order of rank pairs)
    std::vector<std::pair<int, int>> E;
    int pidx = 0;
    for (int a = 0; a < k; ++a)
        for (int b = a + 1; b < k; ++b, ++pidx)
            if ((ecode >> (eb - 1 - pidx)) & 1u) E.push_back({ds[a], ds[b]});
    mapa_status st = fill_decision(t, p, F, S, E, selector, sens, score, d);
    if (st != MAPA_OK) return st;
    *out = d;
    return MAPA_OK;
}

// Topo-aware partitions (reading A21; SPEC select_topo_aware S:337-344,
// "recursive bi-partitioning"): every socket group, recursively halved
// by sorted id (first half = ceil(n/2)) down to single devices, plus the whole
// machine; ordered by size, ties by lowest device id.
void topo_partitions(const mapa_topology *t, uint32_t *part, int32_t *npart) {
    std::vector<std::vector<int>> all;
    std::vector<std::vector<int>> stack(t->sockets.rbegin(), t->sockets.rend());
    while (!stack.empty()) {
        std::vector<int> g = stack.back();
        stack.pop_back();
        std::sort(g.begin(), g.end());
        all.push_back(g);
        if (g.size() > 1) {
            const size_t h = (g.size() + 1) / 2;
            stack.push_back(std::vector<int>(g.begin() + h, g.end()));
            stack.push_back(std::vector<int>(g.begin(), g.begin() + h));
        }
    }
    std::vector<int> whole;
    for (int d = 0; d < t->n; ++d) whole.push_back(d);
    all.push_back(whole);
    std::stable_sort(all.begin(), all.end(), [](const std::vector<int> &a, const std::vector<int> &b) {
        return a.size() != b.size() ? a.size() < b.size() : a.front() < b.front();
    });
    int n = 0;
    for (auto &g : all) {
        if (n >= kMaxParts) break;
        uint32_t m = 0;
        for (int d : g) m |= 1u << d;
        if (n > 0 && part[n - 1] == m) continue;  // a one-socket machine repeats the root
        part[n++] = m;
    }
    *npart = n;
}

mapa_status build_multi(const mapa_topology *t, const mapa_pattern *const *pats, int npats, uint32_t flags,
                        MultiTables *tb) {
    if (npats < 1 || npats > kMaxPats) return fail(MAPA_E_INVALID_ARG, "npats must be 1..16");
    if (t->n > kMaxN) return fail(MAPA_E_UNSUPPORTED, "batch / trace / simulation need N <= 32");
    std::memset(tb, 0, sizeof(*tb));
    fill_devtopo(t, tb->topo);
    topo_partitions(t, tb->part, &tb->npart);
    tb->npats = npats;
    int mmax = 0;
    for (int i = 0; i < npats; ++i)
        if (pats[i]) mmax = std::max(mmax, pats[i]->m);
    tb->xs = pick_xs(mmax);
    int off = 0;
    for (int i = 0; i < npats; ++i) {
        if (!pats[i]) return fail(MAPA_E_INVALID_ARG, "null pattern");
        if (!key_fits(t, pats[i])) return fail(MAPA_E_UNSUPPORTED, "batch / trace patterns need the narrow path (k <= 8)");
        const int n = (int)pats[i]->lut.size();
        if (off + n > kLutCapMulti) return fail(MAPA_E_UNSUPPORTED, "rank tables exceed 4096 entries");
        fill_devpattern(pats[i], (flags & MAPA_F_RAW) != 0, (uint16_t)off, tb->pat[i]);
        std::memcpy(tb->lut + off, pats[i]->lut.data(), n * sizeof(uint16_t));
        off += n;
    }
    return MAPA_OK;
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

const char *mapa_last_error(void) { return g_err.c_str(); }
const char *mapa_version(void) { return "mapa-b200 0.1 (sm_100a)"; }

mapa_status mapa_load_topology(const char *spec, int32_t is_text, mapa_topology **out) {
    if (!spec || !out) return fail(MAPA_E_INVALID_ARG, "null argument");
    mapa_topology *t = new (std::nothrow) mapa_topology();
    if (!t) return fail(MAPA_E_INVALID_ARG, "out of memory");
    if (!is_text) {
        if (!build_builtin(spec, t)) {
            delete t;
            return fail(MAPA_E_INVALID_ARG, std::string("unknown builtin '") + spec +
                                                "'; valid: dgx1v dgx1p summit torus2d16 cubemesh16");
        }
    } else {
        mapa_status st = parse_topology_text(spec, t);
        if (st != MAPA_OK) { delete t; return st; }
    }
    *out = t;
    return MAPA_OK;
}

void mapa_free_topology(mapa_topology *t) {
    if (!t) return;
    for (auto &g : t->graphs) cudaGraphExecDestroy(g.exec);
    for (auto &g : t->many_graphs) cudaGraphExecDestroy(g.exec);
    if (t->d_many) cudaFree(t->d_many);
    if (t->h_many) cudaFreeHost(t->h_many);
    for (auto &pt : t->pair_tabs) cudaFree(pt.d);
    for (auto s2 : t->side) cudaStreamDestroy(s2);
    if (t->cap) cudaStreamDestroy(t->cap);
    if (t->d_stage) cudaFree(t->d_stage);
    if (t->h_stage) cudaFreeHost(t->h_stage);
    if (t->ev_mix) cudaEventSynchronize(t->ev_mix), cudaEventDestroy(t->ev_mix);
    if (t->d_mix) cudaFree(t->d_mix);
    if (t->h_mix) cudaFreeHost(t->h_mix);
    delete t;
}

mapa_status mapa_topology_info(const mapa_topology *t, int32_t *n, int32_t *width, int32_t *bw, uint64_t *busy) {
    if (!t) return fail(MAPA_E_INVALID_ARG, "null topology");
    if (n) *n = t->n;
    if (width) *width = t->width;
    if (busy) *busy = t->busy;
    if (bw)
        for (int u = 0; u < t->n; ++u)
            for (int v = 0; v < t->n; ++v) bw[u * t->n + v] = u == v ? 0 : bw_of(t, u, v);
    return MAPA_OK;
}

mapa_status mapa_claim(mapa_topology *t, uint64_t mask) {
    if (!t) return fail(MAPA_E_INVALID_ARG, "null topology");
    if (mask & ~nmask_of(t->n)) return fail(MAPA_E_ID_RANGE, "device id out of range");
    if (mask & t->busy) return fail(MAPA_E_ALREADY_BUSY, "device already busy");
    t->busy |= mask;
    return MAPA_OK;
}

mapa_status mapa_release(mapa_topology *t, uint64_t mask) {
    if (!t) return fail(MAPA_E_INVALID_ARG, "null topology");
    if (mask & ~nmask_of(t->n)) return fail(MAPA_E_ID_RANGE, "device id out of range");
    if (mask & ~t->busy) return fail(MAPA_E_NOT_BUSY, "releasing a device that is not busy");
    t->busy &= ~mask;
    return MAPA_OK;
}

mapa_status mapa_set_busy(mapa_topology *t, uint64_t busy) {
    if (!t) return fail(MAPA_E_INVALID_ARG, "null topology");
    if (busy & ~nmask_of(t->n)) return fail(MAPA_E_ID_RANGE, "device id out of range");
    t->busy = busy;
    return MAPA_OK;
}

mapa_status mapa_load_pattern(int32_t k, int32_t m, const int32_t *edges, uint32_t flags, mapa_pattern **out) {
    if (!out || m < 0 || (m > 0 && !edges)) return fail(MAPA_E_INVALID_ARG, "bad pattern arguments");
    if (k < 1 || k > kMaxKDeep) return fail(MAPA_E_UNSUPPORTED, "pattern: need 1 <= k <= 16");
    if (m > k * (k - 1) / 2) return fail(MAPA_E_INVALID_ARG, "pattern: more edges than vertex pairs");
    std::vector<std::pair<int, int>> e;
    for (int i = 0; i < m; ++i) e.push_back({edges[2 * i], edges[2 * i + 1]});
    return compile_pattern(k, e, flags, out);
}

mapa_status mapa_make_pattern(int32_t shape, int32_t k, mapa_pattern **out) {
    if (!out) return fail(MAPA_E_INVALID_ARG, "null out");
    if (k < 1 || k > kMaxKDeep) return fail(MAPA_E_UNSUPPORTED, "pattern: need 1 <= k <= 16");
    std::vector<std::pair<int, int>> e;
    const bool ring = shape == MAPA_SHAPE_RING || shape == MAPA_SHAPE_RINGTREE;
    const bool tree = shape == MAPA_SHAPE_TREE || shape == MAPA_SHAPE_RINGTREE;
    if (shape == MAPA_SHAPE_RING && k == 1) return fail(MAPA_E_INVALID_ARG, "Ring requires k >= 2");
    if (shape < 0 || shape > MAPA_SHAPE_EDGELESS) return fail(MAPA_E_INVALID_ARG, "unknown shape");
    std::map<std::pair<int, int>, int> set;
    if (ring) {
        if (k == 2) set[{0, 1}] = 1;
        if (k >= 3)
            for (int i = 0; i < k; ++i) set[{std::min(i, (i + 1) % k), std::max(i, (i + 1) % k)}] = 1;
    }
    if (tree)
        for (int i = 0; i < k; ++i)
            for (int c = 2 * i + 1; c <= 2 * i + 2; ++c)
                if (c < k) set[{i, c}] = 1;
    if (shape == MAPA_SHAPE_FULL)
        for (int a = 0; a < k; ++a)
            for (int b = a + 1; b < k; ++b) set[{a, b}] = 1;
    for (auto &kv : set) e.push_back(kv.first);
    return compile_pattern(k, e, shape == MAPA_SHAPE_EDGELESS ? MAPA_F_ALLOW_DISCONNECTED : 0, out);
}

void mapa_free_pattern(mapa_pattern *p) {
    if (!p) return;
    if (p->clique) mapa_free_pattern(p->clique);
    free_luts(p);
    delete p;
}

mapa_status mapa_get_pattern_info(const mapa_pattern *p, mapa_pattern_info *out) {
    if (!p || !out) return fail(MAPA_E_INVALID_ARG, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->k = p->k;
    out->m = p->m;
    out->aut_order = (int32_t)std::min<uint64_t>(p->aut, 0x7FFFFFFFull);
    out->aut_order64 = p->aut;
    for (int j = 0; j < p->k; ++j) { out->back[j] = p->back[j]; out->lex_src[j] = p->src[j]; }
    for (int e = 0; e < p->m; ++e) { out->edges[e][0] = p->edges[e].first; out->edges[e][1] = p->edges[e].second; }
    return MAPA_OK;
}

double mapa_pred_effbw(int32_t x, int32_t y, int32_t z) { return eq2(x, y, z); }

mapa_status mapa_effbw_rank_table(int32_t m, uint16_t *out) {
    if (m < 0 || m > kMaxEdges || !out) return fail(MAPA_E_INVALID_ARG, "m must be 0..120");
    std::vector<uint16_t> l = rank_table(m);
    std::memcpy(out, l.data(), l.size() * sizeof(uint16_t));
    return MAPA_OK;
}

static mapa_status launch_query_impl(const mapa_topology *t, const mapa_pattern *p, int32_t selector, int32_t sensitive,
                              const mapa_query *d_query, mapa_record *d_record, uint32_t flags, int32_t rank,
                              int32_t world, uint64_t busy_hint, void *stream, bool zero_record);
static mapa_status launch_query_wide_impl(const mapa_topology *t, const mapa_pattern *p, int32_t selector,
                                   int32_t sensitive, const mapa_query64 *d_query, mapa_wide_record *d_record,
                                   uint32_t flags, int32_t rank, int32_t world, uint64_t busy_hint, void *stream,
                                   bool zero_record);

mapa_status mapa_launch_query(const mapa_topology *t, const mapa_pattern *p, int32_t selector,
                                  int32_t sensitive, const mapa_query *d_query, mapa_record *d_record,
                                  uint32_t flags, int32_t rank, int32_t world, uint64_t busy_hint,
                                  void *stream) {
    const NvtxRange nvtx_range_("mapa_launch_query");
    return launch_query_impl(t, p, selector, sensitive, d_query, d_record, flags, rank, world, busy_hint, stream,
                             !(flags & MAPA_F_ZEROED));
}

static mapa_status launch_query_impl(const mapa_topology *t, const mapa_pattern *p, int32_t selector, int32_t sensitive,
                              const mapa_query *d_query, mapa_record *d_record, uint32_t flags, int32_t rank,
                              int32_t world, uint64_t busy_hint, void *stream, bool zero_record) {
    if (!t || !p || !d_query || !d_record) return fail(MAPA_E_INVALID_ARG, "null argument");
    if (t->n > kMaxN) return fail(MAPA_E_UNSUPPORTED, "narrow path needs N <= 32 (use the deep path)");
    if (world < 1 || rank < 0 || rank >= world) return fail(MAPA_E_INVALID_ARG, "bad rank/world");
    if (selector < 0 || selector > 2) return fail(MAPA_E_INVALID_ARG, "bad selector");
    if (!key_fits(t, p))
        return fail(MAPA_E_UNSUPPORTED, "narrow path needs k <= 8 and 15 + W + C(k,2) <= 63 (use the deep path)");
    const int nF = busy_hint == ~0ull ? t->n : __builtin_popcountll(~busy_hint & nmask_of(t->n));
    static_assert(sizeof(SingleTables) < 32000, "kernel parameter block too large");
    SingleTables tb;
    std::memset(&tb, 0, sizeof(tb));
    fill_devtopo(t, tb.topo);
    tb.npats = 1;
    tb.xs = pick_xs(p->m);
    fill_devpattern(p, (flags & MAPA_F_RAW) != 0, 0, tb.pat[0]);
    tb.pre = pair_tables(t, tb.xs, stream);
    // canonical instantiation only when a lex-leader constraint exists (|Aut| > 1
    // and not RAW); otherwise the constraint-free kernel enumerates the same set
    const bool prune = (flags & MAPA_F_PRUNE) && p->k >= 4;
    const int sc = sel_code(selector, sensitive) | (has_constraints(tb.pat[0]) ? 4 : 0) | (prune ? 16 : 0) |
                   (lin16_fits(t, p, sel_code(selector, sensitive), busy_hint, prune ? kLin16Max : kLin16StatMax)
                        ? 32 : 0);
    Plan pl = plan_single(t, p, sc, nF, world);
    if (pl.nlocal >= (1ull << 27)) return fail(MAPA_E_UNSUPPORTED, "too many work items");
    std::memcpy(tb.lut, p->lut.data(), p->lut.size() * sizeof(uint16_t));
    int err = zero_record ? (int)cudaMemsetAsync(d_record, 0, sizeof(mapa_record), (cudaStream_t)stream) : 0;
    if (err) return cuda_fail(err, "cudaMemsetAsync");
    err = launch_single(tb, sc, d_query, d_record, pl.depth, rank, world, pl.chunk, pl.grid, stream);
    if (err) return cuda_fail(err, "esa_single launch");
    return MAPA_OK;
}

mapa_status mapa_launch_queries(mapa_topology *t, const mapa_pattern *const *pats, int32_t npats, int32_t nq,
                                const mapa_query *h_queries, const mapa_query *d_queries, mapa_record *d_records,
                                uint32_t flags, int32_t nstreams, void *stream) {
    const NvtxRange nvtx_range_("mapa_launch_queries");
    if (!t || !pats || nq < 0 || (nq > 0 && (!h_queries || !d_queries || !d_records)) || nstreams < 1 || nstreams > 32)
        return fail(MAPA_E_INVALID_ARG, "bad arguments");
    if (nq == 0) return MAPA_OK;
    cudaStream_t main = (cudaStream_t)stream;
    int err;
    mapa_status sb = bind_device(t);
    if (sb != MAPA_OK) return sb;
    while ((int)t->side.size() < nstreams) {
        cudaStream_t s2;
        if ((err = (int)cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking))) return cuda_fail(err, "cudaStreamCreate");
        t->side.push_back(s2);
    }
    for (int i = 0; i < npats; ++i)  // warm the table cache outside the fork (it may allocate)
        if (pats[i] && key_fits(t, pats[i])) pair_tables(t, pick_xs(pats[i]->m), stream);
    if ((err = (int)cudaMemsetAsync(d_records, 0, (size_t)nq * sizeof(mapa_record), main))) return cuda_fail(err, "memset");
    cudaEvent_t fork, join;
    if ((err = (int)cudaEventCreateWithFlags(&fork, cudaEventDisableTiming))) return cuda_fail(err, "cudaEventCreate");
    if ((err = (int)cudaEventCreateWithFlags(&join, cudaEventDisableTiming))) {  // both before the fork
        cudaEventDestroy(fork);
        return cuda_fail(err, "cudaEventCreate");
    }
    // Small queries (fewer than kMixLeaves leaves) go to ONE batch launch on
    // side stream 0, ordered by code path (k, selector); the others keep a
    // full-GPU single-query launch each, round-robin over the side streams.
    // A single launch costs ~10 us of fixed time (prologue, ramp, drain), more
    // than a small query's work.  Same records either way (max / sum).
    constexpr double kMixLeaves = 4194304.0;
    std::vector<uint32_t> small;
    bool can_batch = npats <= kMaxPats && !(flags & MAPA_F_PRUNE) && t->n <= kMaxN;
    for (int i = 0; i < npats && can_batch; ++i) can_batch = pats[i] && key_fits(t, pats[i]);
    std::vector<char> is_small((size_t)nq, 0);
    for (int i = 0; i < nq; ++i) {
        const mapa_query &q = h_queries[i];
        if (q.pattern >= (uint32_t)npats || !pats[q.pattern]) {
            cudaEventDestroy(fork);
            cudaEventDestroy(join);
            return fail(MAPA_E_INVALID_ARG, "query pattern index out of range");
        }
        if (!can_batch) continue;
        const mapa_pattern *p = pats[q.pattern];
        const int nf = __builtin_popcountll(~(uint64_t)q.busy & nmask_of(t->n));
        double w = 1.0;
        for (int j = 0; j < p->k; ++j) w *= (double)std::max(0, nf - j);
        if (!(flags & MAPA_F_RAW)) w /= (double)p->aut;
        if (w < kMixLeaves && q.selector >= 0 && q.selector <= 2) { is_small[(size_t)i] = 1; small.push_back((uint32_t)i); }
    }
    if (small.size() < 2) {
        small.clear();
        std::fill(is_small.begin(), is_small.end(), 0);
    }
    cudaEventRecord(fork, main);
    for (int s2 = 0; s2 < nstreams; ++s2) cudaStreamWaitEvent(t->side[s2], fork, 0);
    mapa_status st = MAPA_OK;
    if (!small.empty()) {
        static thread_local MultiTables *tbp = nullptr;
        if (!tbp) tbp = new MultiTables();
        st = build_multi(t, pats, npats, flags, tbp);
        const size_t bytes = 64 + 4 * small.size();
        if (st == MAPA_OK && bytes > t->mix_cap) {
            if (t->ev_mix) cudaEventSynchronize(t->ev_mix);
            if (t->d_mix) cudaFree(t->d_mix);
            if (t->h_mix) cudaFreeHost(t->h_mix);
            t->d_mix = t->h_mix = nullptr;
            t->mix_cap = 0;
            if ((err = (int)cudaMalloc(&t->d_mix, bytes)) || (err = (int)cudaMallocHost(&t->h_mix, bytes)))
                st = cuda_fail(err, "cudaMalloc (query batch)");
            else
                t->mix_cap = bytes;
        }
        if (st == MAPA_OK && !t->ev_mix && (err = (int)cudaEventCreateWithFlags(&t->ev_mix, cudaEventDisableTiming)))
            st = cuda_fail(err, "cudaEventCreate");
        if (st == MAPA_OK) {
            cudaEventSynchronize(t->ev_mix);  // the previous call's copy out of h_mix is done
            std::stable_sort(small.begin(), small.end(), [&](uint32_t a, uint32_t b) {
                const mapa_query &qa = h_queries[a], &qb = h_queries[b];
                const int ka = pats[qa.pattern]->k * 4 + sel_code(qa.selector, qa.sensitive);
                const int kb = pats[qb.pattern]->k * 4 + sel_code(qb.selector, qb.sensitive);
                return ka < kb;
            });
            std::memcpy((char *)t->h_mix + 64, small.data(), 4 * small.size());
            cudaStream_t s0 = t->side[0];
            int sm = device_sm_count();
            if (sm <= 0) sm = 148;
            const int canon = multi_has_constraints(*tbp);
            const int grid = sm * max_blocks_per_sm_batch(t->width, canon, tbp->npats, tbp->xs);
            if ((err = (int)cudaMemsetAsync(t->d_mix, 0, 64, s0)) ||
                (err = (int)cudaMemcpyAsync((char *)t->d_mix + 64, (char *)t->h_mix + 64, 4 * small.size(),
                                            cudaMemcpyHostToDevice, s0)) ||
                (err = (int)cudaEventRecord(t->ev_mix, s0)) ||
                (err = launch_batch(*tbp, canon, (int64_t)small.size(), d_queries, d_records, (uint32_t *)t->d_mix,
                                    (const uint32_t *)((char *)t->d_mix + 64), grid, (void *)s0)))
                st = cuda_fail(err, "query batch launch");
        }
    }
    int nb = 0;
    for (int i = 0; i < nq && st == MAPA_OK; ++i) {
        if (is_small[(size_t)i]) continue;
        const mapa_query &q = h_queries[i];
        if (q.selector < 0 || q.selector > 2) { st = fail(MAPA_E_INVALID_ARG, "bad selector"); break; }
        st = launch_query_impl(t, pats[q.pattern], q.selector, q.sensitive, d_queries + i, d_records + i, flags, 0, 1,
                               q.busy, (void *)t->side[(nb++ + (small.empty() ? 0 : 1)) % nstreams], false);
    }
    for (int s2 = 0; s2 < nstreams; ++s2) {  // join: every side stream's work before `main` continues
        cudaEventRecord(join, t->side[s2]);
        cudaStreamWaitEvent(main, join, 0);
    }
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    return st;
}

mapa_status mapa_reduce_records(const mapa_record *records, int32_t n, mapa_record *out) {
    if (!records || !out || n < 1) return fail(MAPA_E_INVALID_ARG, "bad records");
    mapa_record r;
    std::memset(&r, 0, sizeof(r));
    for (int i = 0; i < n; ++i) {
        r.key = std::max(r.key, records[i].key);
        r.leaves += records[i].leaves;
        r.status |= records[i].status;
    }
    *out = r;
    return MAPA_OK;
}

mapa_status mapa_decode(const mapa_topology *t, const mapa_pattern *p, uint64_t busy, int32_t selector,
                        int32_t sens, uint32_t flags, const mapa_record *record, mapa_decision *out) {
    if (!t || !p || !record || !out) return fail(MAPA_E_INVALID_ARG, "null argument");
    return decode_record(t, p, busy, selector, sens, flags, record, out);
}

mapa_status mapa_launch_query_wide(const mapa_topology *t, const mapa_pattern *p, int32_t selector,
                                   int32_t sensitive, const mapa_query64 *d_query, mapa_wide_record *d_record,
                                   uint32_t flags, int32_t rank, int32_t world, uint64_t busy_hint, void *stream) {
    const NvtxRange nvtx_range_("mapa_launch_query_wide");
    return launch_query_wide_impl(t, p, selector, sensitive, d_query, d_record, flags, rank, world, busy_hint,
                                  stream, !(flags & MAPA_F_ZEROED));
}

static mapa_status launch_query_wide_impl(const mapa_topology *t, const mapa_pattern *p, int32_t selector,
                                   int32_t sensitive, const mapa_query64 *d_query, mapa_wide_record *d_record,
                                   uint32_t flags, int32_t rank, int32_t world, uint64_t busy_hint, void *stream,
                                   bool zero_record) {
    if (!t || !p || !d_query || !d_record) return fail(MAPA_E_INVALID_ARG, "null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(MAPA_E_INVALID_ARG, "bad rank/world");
    if (selector < 0 || selector > 2) return fail(MAPA_E_INVALID_ARG, "bad selector");
    if (busy_hint & ~nmask_of(t->n)) return fail(MAPA_E_INVALID_ARG, "deep path needs busy_hint = the query's busy mask");
    const int nF = __builtin_popcountll(~busy_hint & nmask_of(t->n));
    cudaStream_t st = (cudaStream_t)stream;
    int err = zero_record ? (int)cudaMemsetAsync(d_record, 0, sizeof(mapa_wide_record), st) : 0;
    if (err) return cuda_fail(err, "cudaMemsetAsync");
    if (p->k > nF) return MAPA_OK;  // no capacity: the zeroed record says so (key 0)
    static_assert(sizeof(DeepTables) < 32000, "kernel parameter block too large");
    mapa_topology *tm = const_cast<mapa_topology *>(t);  // plan cache (immutable inputs)
    const bool canon_req = !(flags & MAPA_F_RAW);
    const uint64_t key[3] = {p->uid, (uint64_t)sel_code(selector, sensitive) | ((uint64_t)canon_req << 3) |
                                         ((uint64_t)((flags & MAPA_F_PRUNE) != 0) << 4),
                             (uint64_t)nF | ((uint64_t)t->n << 8) | ((uint64_t)world << 16)};
    mapa_topology::DeepPlanEntry *e = nullptr;
    for (auto &x : tm->deep_plans)
        if (x->key[0] == key[0] && x->key[1] == key[1] && x->key[2] == key[2]) { e = x.get(); break; }
    mapa_status s;
    if (!e) {
        std::unique_ptr<mapa_topology::DeepPlanEntry> ne(new (std::nothrow) mapa_topology::DeepPlanEntry());
        if (!ne) return fail(MAPA_E_INVALID_ARG, "out of memory");
        DeepPlan pl{};
        s = plan_deep(t, p, selector, sensitive, flags, nF, world, &ne->tb, &pl);
        if (s != MAPA_OK) return s;
        std::memcpy(ne->key, key, sizeof(key));
        ne->sc = pl.sc; ne->depth = pl.depth; ne->stripe = pl.stripe; ne->grid = pl.grid;
        if (tm->deep_plans.size() >= 16) {  // evict the least recently used
            auto lru = std::min_element(tm->deep_plans.begin(), tm->deep_plans.end(),
                                        [](const std::unique_ptr<mapa_topology::DeepPlanEntry> &a2,
                                           const std::unique_ptr<mapa_topology::DeepPlanEntry> &b2) {
                                            return a2->tick < b2->tick;
                                        });
            tm->deep_plans.erase(lru);
        }
        tm->deep_plans.push_back(std::move(ne));
        e = tm->deep_plans.back().get();
    }
    e->tick = ++tm->tick;
    const uint16_t *d_lut = nullptr;
    if (sel_code(selector, sensitive) == SEL_SENS && (s = upload_lut(p, &d_lut)) != MAPA_OK) return s;
    err = launch_deep(e->tb, e->sc, d_lut, d_query, d_record, e->depth, rank, world,
                      e->stripe, e->grid, stream);
    if (err) return cuda_fail(err, "esa_deep launch");
    return MAPA_OK;
}

mapa_status mapa_reduce_wide_records(const mapa_wide_record *records, int32_t n, mapa_wide_record *out) {
    if (!records || !out || n < 1) return fail(MAPA_E_INVALID_ARG, "bad records");
    mapa_wide_record r;
    std::memset(&r, 0, sizeof(r));
    for (int i = 0; i < n; ++i) {
        const mapa_wide_record &q = records[i];
        const uint64_t a[4] = {q.score, q.set, q.ecode_hi, q.ecode_lo};
        const uint64_t b[4] = {r.score, r.set, r.ecode_hi, r.ecode_lo};
        if (q.set && std::lexicographical_compare(b, b + 4, a, a + 4)) {
            r.score = q.score; r.set = q.set; r.ecode_hi = q.ecode_hi; r.ecode_lo = q.ecode_lo;
        }
        r.leaves += q.leaves;
        r.status |= q.status;
    }
    *out = r;
    return MAPA_OK;
}

mapa_status mapa_decode_wide(const mapa_topology *t, const mapa_pattern *p, uint64_t busy, int32_t selector,
                             int32_t sens, uint32_t flags, const mapa_wide_record *record, mapa_decision *out) {
    if (!t || !p || !record || !out) return fail(MAPA_E_INVALID_ARG, "null argument");
    return decode_wide(t, p, busy, selector, sens, flags, record, out);
}

// Is there a bijection sigma: V(P) -> {0..k-1} with, for every decided rank
// pair p < np (lex order), [sigma^-1 of its ranks adjacent in P] == bit p?
// Backtracking over ranks 0..k-1: rank i takes an unused pattern vertex whose
// adjacency to the vertices of ranks j < i matches every decided pair (j, i),
// and every placed rank's decided 1s / 0s towards the unplaced ranks must fit
// its unplaced neighbours / non-neighbours (counting prune).  `budget` bounds
// the nodes visited; -1 = budget exhausted (undecided).
int labelling_exists(const mapa_pattern *p, const std::vector<int> &pidx, const uint8_t *bit, int np, int i,
                     int *inv, uint32_t used, long long &budget) {
    const int k = p->k;
    if (i == k) return 1;
    for (int u = 0; u < k; ++u) {
        if ((used >> u) & 1u) continue;
        if (--budget < 0) return -1;
        bool ok = true;
        for (int j = 0; j < i && ok; ++j) {
            const int q = pidx[j * k + i];
            if (q < np) ok = (((p->adj[inv[j]] >> u) & 1u) != 0) == (bit[q] != 0);
        }
        if (!ok) continue;
        inv[i] = u;
        const uint32_t used2 = used | (1u << u);
        const int rest = k - i - 1;
        for (int j = 0; j <= i && ok; ++j) {  // counting prune on every placed rank
            int need1 = 0, need0 = 0;
            for (int x = i + 1; x < k; ++x) {
                const int q = pidx[j * k + x];
                if (q < np) (bit[q] ? need1 : need0)++;
            }
            const int nb = __builtin_popcount((uint32_t)p->adj[inv[j]] & ~used2 & ((1u << k) - 1u));
            ok = need1 <= nb && need0 <= rest - nb;
        }
        if (!ok) continue;
        const int r = labelling_exists(p, pidx, bit, np, i + 1, inv, used2, budget);
        if (r != 0) return r;
    }
    return 0;
}

// The pattern's lex-smallest used-edge list over rank pairs, as the 128-bit
// edge code (bit C(k,2)-1-p for the p-th rank pair in lex order): maximise the
// code bit by bit -- keep bit p set iff some labelling still satisfies every
// decided pair (the greedy is exact for a lexicographic maximum).  Weight
// independent: the tie-break among equal-score mappings of one device set.
// Returns false if the search budget ran out (the caller then searches
// exhaustively).
bool lexmin_labelling(const mapa_pattern *p, uint64_t out[2]) {
    const int k = p->k, eb = k * (k - 1) / 2;
    std::vector<int> pidx((size_t)k * k, 0);
    int q = 0;
    for (int a2 = 0; a2 < k; ++a2)
        for (int b2 = a2 + 1; b2 < k; ++b2) pidx[a2 * k + b2] = pidx[b2 * k + a2] = q++;
    std::vector<uint8_t> bit(eb, 0);
    int inv[kMaxKDeep];
    int ones = 0;
    long long budget = 20000000;  // nodes over all feasibility checks
    for (int p2 = 0; p2 < eb; ++p2) {
        bit[p2] = 1;
        if (ones < p->m) {
            const int r = labelling_exists(p, pidx, bit.data(), p2 + 1, 0, inv, 0u, budget);
            if (r < 0) return false;
            if (r == 1) {
                ++ones;
                continue;
            }
        }
        bit[p2] = 0;
    }
    out[0] = out[1] = 0;
    for (int p2 = 0; p2 < eb; ++p2)
        if (bit[p2]) {
            const int qq = eb - 1 - p2;
            if (qq >= 64) out[0] |= 1ull << (qq - 64);
            else out[1] |= 1ull << qq;
        }
    return true;
}

// Preserve-insensitive on the deep path with MAPA_F_PRUNE: Eq. 3 depends on
// the device set only, so (1) the best set -- max PreservedBW, ties to the
// lex-smallest set -- is the decision of the full-k pattern (one canonical
// leaf per k-subset), and (2) every mapping of that set scores the same, so
// the winning used-edge list is the pattern's lex-smallest one over rank
// pairs, which does not depend on the weights: computed once per pattern on
// the host (lexmin_labelling) and cached.  Same decision as the exhaustive
// search (tests); leaves = the set search's leaves.
static mapa_status allocate_insens_sets(mapa_topology *t, const mapa_pattern *pc, int selector, uint32_t flags,
                                        void *stream, mapa_decision *out) {
    mapa_pattern *p = const_cast<mapa_pattern *>(pc);  // caches of immutable derived data
    const int k = p->k;
    mapa_status s;
    if (!p->have_ecode_min) {
        if (!lexmin_labelling(p, p->ecode_min))  // budget exhausted: exhaustive deep search instead
            return mapa_allocate(t, pc, selector, 0, flags & ~(uint32_t)MAPA_F_PRUNE, stream, out);
        p->have_ecode_min = true;
    }
    if (selector == MAPA_SEL_BASELINE) {
        // constant score: the k lowest free ids, the lex-smallest labelling
        mapa_wide_record rec;
        std::memset(&rec, 0, sizeof(rec));
        uint64_t free = ~t->busy & nmask_of(t->n);
        for (int i = 0; i < k; ++i) {
            const int d = __builtin_ctzll(free);
            free &= free - 1;
            rec.set |= 1ull << (63 - d);
        }
        rec.ecode_hi = p->ecode_min[0];
        rec.ecode_lo = p->ecode_min[1];
        mapa_decision d;
        if ((s = decode_wide(t, p, t->busy, MAPA_SEL_BASELINE, 0, flags & ~(uint32_t)MAPA_F_PRUNE, &rec, &d)) != MAPA_OK)
            return s;
        uint64_t perm = 1;
        const int nf = __builtin_popcountll(~t->busy & nmask_of(t->n));
        for (int i = 0; i < k; ++i) perm *= (uint64_t)std::max(0, nf - i);
        d.raw_embeddings = perm;
        d.distinct_matches = perm / p->aut;
        d.leaves_scored = 0;
        if (flags & MAPA_F_COMMIT) t->busy |= d.device_mask;
        *out = d;
        return MAPA_OK;
    }
    if (!p->clique) {
        std::vector<std::pair<int, int>> all;
        for (int a = 0; a < k; ++a)
            for (int b = a + 1; b < k; ++b) all.push_back({a, b});
        if ((s = compile_pattern(k, all, 0, &p->clique)) != MAPA_OK) return s;
    }
    // canonical even under MAPA_F_RAW: the clique has one orbit per set, so the
    // decision is the same and RAW would enumerate k! permutations of each set
    const uint32_t sub = flags & ~(uint32_t)(MAPA_F_COMMIT | MAPA_F_PRUNE | MAPA_F_RAW);
    mapa_decision dc;
    if ((s = mapa_allocate(t, p->clique, MAPA_SEL_PRESERVE, 0, sub, stream, &dc)) != MAPA_OK) return s;
    const uint64_t extra = 0;
    mapa_wide_record rec;
    std::memset(&rec, 0, sizeof(rec));
    rec.score = (uint64_t)(uint32_t)dc.score;
    for (int d = 0; d < 64; ++d)
        if ((dc.device_mask >> d) & 1ull) rec.set |= 1ull << (63 - d);
    rec.ecode_hi = p->ecode_min[0];
    rec.ecode_lo = p->ecode_min[1];
    rec.leaves = dc.leaves_scored + extra;
    mapa_decision d;
    if ((s = decode_wide(t, p, t->busy, MAPA_SEL_PRESERVE, 0, flags & ~(uint32_t)MAPA_F_PRUNE, &rec, &d)) != MAPA_OK)
        return s;
    uint64_t perm = 1;  // counts: the closed forms (the search scored sets, not embeddings)
    const int nf = __builtin_popcountll(~t->busy & nmask_of(t->n));
    for (int i = 0; i < k; ++i) perm *= (uint64_t)std::max(0, nf - i);
    d.raw_embeddings = perm;
    d.distinct_matches = perm / p->aut;
    if (flags & MAPA_F_COMMIT) t->busy |= d.device_mask;
    *out = d;
    return MAPA_OK;
}

mapa_status mapa_allocate(mapa_topology *t, const mapa_pattern *p, int32_t selector, int32_t sens,
                          uint32_t flags, void *stream, mapa_decision *out) {
    const NvtxRange nvtx_range_("mapa_allocate");
    if (!t || !p || !out) return fail(MAPA_E_INVALID_ARG, "null argument");
    if (selector < 0 || selector > 2) return fail(MAPA_E_INVALID_ARG, "bad selector");
    const bool deep = (flags & MAPA_F_DEEP) || !key_fits(t, p);
    const uint64_t F = ~t->busy & nmask_of(t->n);
    if (p->k > __builtin_popcountll(F)) {
        std::memset(out, 0, sizeof(*out));
        out->status = MAPA_NO_CAPACITY;
        out->k = p->k;
        out->m = p->m;
        return MAPA_NO_CAPACITY;
    }
    if (deep && (flags & MAPA_F_PRUNE) && p->k >= 2 &&
        ((selector == MAPA_SEL_PRESERVE && !sens) || selector == MAPA_SEL_BASELINE))
        return allocate_insens_sets(t, p, selector, flags, stream, out);
    int err;
    mapa_status sb = bind_device(t);
    if (sb != MAPA_OK) return sb;
    if (!t->d_stage) {
        if ((err = (int)cudaMalloc(&t->d_stage, 128))) return cuda_fail(err, "cudaMalloc");
    }
    if (!t->h_stage) {
        if ((err = (int)cudaMallocHost(&t->h_stage, 192))) return cuda_fail(err, "cudaMallocHost");
        std::memset(t->h_stage, 0, 192);
    }
    // staging: host [0,16) query (mapa_query narrow / mapa_query64 deep), [64,128)
    // a zero record (never written), [128,192) the result; ONE 128-B H2D copy
    // stages the query and zeroes the device record (device [0,16) / [64,128))
    void *hq = t->h_stage, *dq = t->d_stage;
    void *hr = (char *)t->h_stage + 128;
    void *dr = (char *)t->d_stage + 64;
    if (deep) {
        mapa_query64 *q = (mapa_query64 *)hq;
        q->busy = t->busy;
        q->selector = selector;
        q->sensitive = sens;
    } else {
        mapa_query *q = (mapa_query *)hq;
        q->busy = (uint32_t)t->busy;
        q->pattern = 0;
        q->selector = selector;
        q->sensitive = sens;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t rbytes = deep ? sizeof(mapa_wide_record) : sizeof(mapa_record);
    const uint32_t lflags = flags;
    // the sequence issued on stream `s2`
    auto issue = [&](cudaStream_t s2) -> mapa_status {
        int e2;
        if ((e2 = (int)cudaMemcpyAsync(dq, hq, 128, cudaMemcpyHostToDevice, s2))) return cuda_fail(e2, "H2D query");
        mapa_status s3 = deep ? launch_query_wide_impl(t, p, selector, sens, (const mapa_query64 *)dq,
                                                       (mapa_wide_record *)dr, lflags, 0, 1, t->busy, (void *)s2, false)
                              : launch_query_impl(t, p, selector, sens, (const mapa_query *)dq, (mapa_record *)dr,
                                                  lflags, 0, 1, t->busy, (void *)s2, false);
        if (s3 != MAPA_OK) return s3;
        if ((e2 = (int)cudaMemcpyAsync(hr, dr, rbytes, cudaMemcpyDeviceToHost, s2))) return cuda_fail(e2, "D2H record");
        return MAPA_OK;
    };
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t key[3] = {p->uid, (uint64_t)selector | ((uint64_t)(sens != 0) << 2) | ((uint64_t)deep << 3) |
                                         ((uint64_t)lflags << 8),
                             (uint64_t)__builtin_popcountll(F) | ((uint64_t)dev << 8)};
    cudaGraphExec_t exec = nullptr;
    for (auto &g : t->graphs)
        if (g.key[0] == key[0] && g.key[1] == key[1] && g.key[2] == key[2]) { exec = g.exec; g.tick = ++t->tick; break; }
    if (!exec) {
        // first call for this key: capture the sequence on a private stream
        if (!deep) pair_tables(t, pick_xs(p->m), stream);  // cudaMalloc / sync copy: not inside the capture
        if (deep && sel_code(selector, sens) == SEL_SENS) {
            const uint16_t *d_lut = nullptr;
            mapa_status su = upload_lut(p, &d_lut);  // synchronous: not inside the capture
            if (su != MAPA_OK) return su;
        }
        if (!t->cap && (err = (int)cudaStreamCreateWithFlags(&t->cap, cudaStreamNonBlocking)))
            return cuda_fail(err, "cudaStreamCreate");
        if ((err = (int)cudaStreamBeginCapture(t->cap, cudaStreamCaptureModeRelaxed))) return cuda_fail(err, "capture");
        const mapa_status sc = issue(t->cap);
        cudaGraph_t graph = nullptr;
        const int ec = (int)cudaStreamEndCapture(t->cap, &graph);
        if (sc != MAPA_OK) { if (graph) cudaGraphDestroy(graph); return sc; }
        if (ec) return cuda_fail(ec, "cudaStreamEndCapture");
        err = (int)cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (err) return cuda_fail(err, "cudaGraphInstantiate");
        if (t->graphs.size() >= 32) {  // evict the least recently used
            auto lru = std::min_element(t->graphs.begin(), t->graphs.end(),
                                        [](const GraphEntry &a2, const GraphEntry &b2) { return a2.tick < b2.tick; });
            cudaGraphExecDestroy(lru->exec);
            t->graphs.erase(lru);
        }
        t->graphs.push_back({{key[0], key[1], key[2]}, exec, ++t->tick});
    }
    if ((err = (int)cudaGraphLaunch(exec, st))) return cuda_fail(err, "cudaGraphLaunch");
    mapa_status s = MAPA_OK;
    if ((err = (int)cudaStreamSynchronize(st))) return cuda_fail(err, "cudaStreamSynchronize");
    mapa_decision d;
    if (deep)
        s = decode_wide(t, p, t->busy, selector, sens, flags, (const mapa_wide_record *)hr, &d);
    else
        s = decode_record(t, p, t->busy, selector, sens, flags, (const mapa_record *)hr, &d);
    if (s < 0) return s;
    if (s == MAPA_OK && (flags & MAPA_F_COMMIT)) t->busy |= d.device_mask;
    *out = d;
    return s;
}

mapa_status mapa_allocate_many(mapa_topology *t, const mapa_pattern *const *pats, int32_t nq, const int32_t *selector,
                               const int32_t *sensitive, uint32_t flags, void *stream, mapa_decision *out) {
    const NvtxRange nvtx_range_("mapa_allocate_many");
    if (!t || nq < 1 || nq > 32 || !pats || !selector || !sensitive || !out)
        return fail(MAPA_E_INVALID_ARG, "bad allocate_many arguments (1 <= nq <= 32)");
    if (flags & MAPA_F_COMMIT) return fail(MAPA_E_INVALID_ARG, "allocate_many never commits (independent queries)");
    for (int i = 0; i < nq; ++i)
        if (!pats[i] || selector[i] < 0 || selector[i] > 2) return fail(MAPA_E_INVALID_ARG, "bad query " + std::to_string(i));
    mapa_status sb = bind_device(t);
    if (sb != MAPA_OK) return sb;
    const uint64_t F = ~t->busy & nmask_of(t->n);
    const int nf = __builtin_popcountll(F);
    int err;
    if (nq > t->many_cap) {
        if (t->d_many) cudaFree(t->d_many);
        if (t->h_many) cudaFreeHost(t->h_many);
        t->d_many = t->h_many = nullptr;
        t->many_cap = 0;
        for (auto &g : t->many_graphs) cudaGraphExecDestroy(g.exec);
        t->many_graphs.clear();  // they hold the old staging pointers
        if ((err = (int)cudaMalloc(&t->d_many, 128 * (size_t)32)) || (err = (int)cudaMallocHost(&t->h_many, 256 * (size_t)32)))
            return cuda_fail(err, "cudaMalloc (allocate_many)");
        std::memset(t->h_many, 0, 256 * 32);
        t->many_cap = 32;
    }
    // staging: host [128 i, 128 i + 16) query i, [128 i + 64, 128 i + 128) a zero
    // record; ONE H2D copy of nq x 128 B stages every query and zeroes every
    // device record; the records come back in one D2H copy into [128 nq, ...)
    std::vector<char> deep(nq);
    for (int i = 0; i < nq; ++i) {
        deep[i] = (flags & MAPA_F_DEEP) || !key_fits(t, pats[i]);
        char *h = (char *)t->h_many + 128 * i;
        std::memset(h, 0, 128);
        if (deep[i]) {
            mapa_query64 *q = (mapa_query64 *)h;
            q->busy = t->busy;
            q->selector = selector[i];
            q->sensitive = sensitive[i];
        } else {
            mapa_query *q = (mapa_query *)h;
            q->busy = (uint32_t)t->busy;
            q->selector = selector[i];
            q->sensitive = sensitive[i];
        }
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::vector<uint64_t> key;
    key.push_back((uint64_t)nq | ((uint64_t)flags << 8) | ((uint64_t)nf << 40) | ((uint64_t)dev << 48));
    for (int i = 0; i < nq; ++i) {
        key.push_back(pats[i]->uid);
        key.push_back((uint64_t)selector[i] | ((uint64_t)(sensitive[i] != 0) << 2) | ((uint64_t)deep[i] << 3));
    }
    cudaGraphExec_t exec = nullptr;
    for (auto &g : t->many_graphs)
        if (g.key == key) { exec = g.exec; g.tick = ++t->tick; break; }
    if (!exec) {
        // warm every cache that allocates or copies synchronously, outside the capture
        for (int i = 0; i < nq; ++i) {
            if (!deep[i]) pair_tables(t, pick_xs(pats[i]->m), stream);
            if (deep[i] && sel_code(selector[i], sensitive[i]) == SEL_SENS) {
                const uint16_t *d_lut = nullptr;
                mapa_status su = upload_lut(pats[i], &d_lut);
                if (su != MAPA_OK) return su;
            }
        }
        if (!t->cap && (err = (int)cudaStreamCreateWithFlags(&t->cap, cudaStreamNonBlocking)))
            return cuda_fail(err, "cudaStreamCreate");
        while ((int)t->side.size() < nq) {
            cudaStream_t s2;
            if ((err = (int)cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking))) return cuda_fail(err, "cudaStreamCreate");
            t->side.push_back(s2);
        }
        cudaEvent_t ev[2];
        if ((err = (int)cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming))) return cuda_fail(err, "cudaEventCreate");
        if ((err = (int)cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming))) {
            cudaEventDestroy(ev[0]);
            return cuda_fail(err, "cudaEventCreate");
        }
        if ((err = (int)cudaStreamBeginCapture(t->cap, cudaStreamCaptureModeRelaxed))) {
            cudaEventDestroy(ev[0]);
            cudaEventDestroy(ev[1]);
            return cuda_fail(err, "capture");
        }
        // one H2D copy, then the nq launches as parallel branches (their
        // prologues and tails overlap), then one D2H copy
        mapa_status sc = MAPA_OK;
        if ((err = (int)cudaMemcpyAsync(t->d_many, t->h_many, 128 * (size_t)nq, cudaMemcpyHostToDevice, t->cap)))
            sc = cuda_fail(err, "H2D queries");
        cudaEventRecord(ev[0], t->cap);
        for (int i = 0; i < nq && sc == MAPA_OK; ++i) {
            cudaStream_t s2 = t->side[i];
            cudaStreamWaitEvent(s2, ev[0], 0);
            char *dq = (char *)t->d_many + 128 * i, *dr = dq + 64;
            sc = deep[i] ? launch_query_wide_impl(t, pats[i], selector[i], sensitive[i], (const mapa_query64 *)dq,
                                                  (mapa_wide_record *)dr, flags, 0, 1, t->busy, (void *)s2, false)
                         : launch_query_impl(t, pats[i], selector[i], sensitive[i], (const mapa_query *)dq,
                                             (mapa_record *)dr, flags, 0, 1, t->busy, (void *)s2, false);
            cudaEventRecord(ev[1], s2);
            cudaStreamWaitEvent(t->cap, ev[1], 0);
        }
        // the nq records (64 B each, pitch 128 on the device) back in one 2-D copy
        if (sc == MAPA_OK && (err = (int)cudaMemcpy2DAsync((char *)t->h_many + 128 * 32, 64, (char *)t->d_many + 64, 128,
                                                           64, (size_t)nq, cudaMemcpyDeviceToHost, t->cap)))
            sc = cuda_fail(err, "D2H records");
        cudaGraph_t graph = nullptr;
        const int ec = (int)cudaStreamEndCapture(t->cap, &graph);
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        if (sc != MAPA_OK) { if (graph) cudaGraphDestroy(graph); return sc; }
        if (ec) return cuda_fail(ec, "cudaStreamEndCapture");
        err = (int)cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (err) return cuda_fail(err, "cudaGraphInstantiate");
        if (t->many_graphs.size() >= 16) {
            auto lru = std::min_element(t->many_graphs.begin(), t->many_graphs.end(),
                                        [](const ManyEntry &a2, const ManyEntry &b2) { return a2.tick < b2.tick; });
            cudaGraphExecDestroy(lru->exec);
            t->many_graphs.erase(lru);
        }
        t->many_graphs.push_back({key, exec, ++t->tick});
    }
    cudaStream_t st = (cudaStream_t)stream;
    if ((err = (int)cudaGraphLaunch(exec, st))) return cuda_fail(err, "cudaGraphLaunch");
    if ((err = (int)cudaStreamSynchronize(st))) return cuda_fail(err, "cudaStreamSynchronize");
    std::vector<mapa_decision> dec(nq);
    for (int i = 0; i < nq; ++i) {
        const char *hr = (const char *)t->h_many + 128 * 32 + 64 * i;
        mapa_status s = deep[i] ? decode_wide(t, pats[i], t->busy, selector[i], sensitive[i], flags,
                                              (const mapa_wide_record *)hr, &dec[i])
                                : decode_record(t, pats[i], t->busy, selector[i], sensitive[i], flags,
                                                (const mapa_record *)hr, &dec[i]);
        if (s < 0) return s;
    }
    std::memcpy(out, dec.data(), sizeof(mapa_decision) * (size_t)nq);
    return MAPA_OK;
}

mapa_status mapa_allocate_batch(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats,
                                int64_t nq, const mapa_query *d_queries, mapa_record *d_results,
                                void *d_scratch, uint32_t flags, void *stream) {
    const NvtxRange nvtx_range_("mapa_allocate_batch");
    if (!t || !pats || (nq > 0 && (!d_queries || !d_results || !d_scratch)) || nq < 0)
        return fail(MAPA_E_INVALID_ARG, "null argument");
    if (flags & MAPA_F_PRUNE) return fail(MAPA_E_UNSUPPORTED, "MAPA_F_PRUNE is single-query only");
    static thread_local MultiTables *tbp = nullptr;  // ~10 KB: keep off the stack
    if (!tbp) tbp = new MultiTables();
    mapa_status s = build_multi(t, pats, npats, flags, tbp);
    if (s != MAPA_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    int err;
    if (nq == 0) return MAPA_OK;
    if ((err = (int)cudaMemsetAsync(d_results, 0, (size_t)nq * sizeof(mapa_record), st))) return cuda_fail(err, "memset");
    // scratch: [0,64) slot counter, [64,192) bucket counts, [192,320) bucket
    // cursors, [512, 512 + 4 nq) the query order (bucketed by code path)
    if ((err = (int)cudaMemsetAsync(d_scratch, 0, 512, st))) return cuda_fail(err, "memset");
    uint32_t *perm = nullptr;
    if (nq < (1ll << 32) && tbp->npats > 1) {  // one pattern: <= 4 code paths, nothing to gain
        BucketKeys bk{};
        bk.npats = tbp->npats;
        for (int i = 0; i < tbp->npats; ++i) bk.k[i] = tbp->pat[i].k;
        char *sc = (char *)d_scratch;
        perm = (uint32_t *)(sc + 512);
        if ((err = launch_bucket(bk, nq, d_queries, (unsigned int *)(sc + 64), (unsigned int *)(sc + 192), perm,
                                 stream)))
            return cuda_fail(err, "bucket launch");
    }
    int sm = device_sm_count();
    if (sm <= 0) sm = 148;
    const int canon = multi_has_constraints(*tbp);
    const int grid = sm * max_blocks_per_sm_batch(t->width, canon, tbp->npats, tbp->xs);
    err = launch_batch(*tbp, canon, nq, d_queries, d_results, (uint32_t *)d_scratch, perm, grid, stream);
    if (err) return cuda_fail(err, "esa_batch launch");
    return MAPA_OK;
}

mapa_status mapa_trace_replay(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats,
                              int32_t ntraces, int32_t nops, const mapa_trace_op *d_ops, int32_t njobs,
                              const mapa_query *d_jobs, uint64_t *d_keys, uint32_t flags, void *stream) {
    const NvtxRange nvtx_range_("mapa_trace_replay");
    if (!t || !pats || ntraces < 0 || nops < 0 || njobs < 0) return fail(MAPA_E_INVALID_ARG, "bad argument");
    if (flags & MAPA_F_PRUNE) return fail(MAPA_E_UNSUPPORTED, "MAPA_F_PRUNE is single-query only");
    if (ntraces == 0) return MAPA_OK;
    if (!d_ops || !d_jobs || !d_keys) return fail(MAPA_E_INVALID_ARG, "null device buffer");
    static thread_local MultiTables *tbp = nullptr;
    if (!tbp) tbp = new MultiTables();
    mapa_status s = build_multi(t, pats, npats, flags, tbp);
    if (s != MAPA_OK) return s;
    int err = (int)cudaMemsetAsync(d_keys, 0, (size_t)ntraces * njobs * sizeof(uint64_t), (cudaStream_t)stream);
    if (err) return cuda_fail(err, "memset");
    err = launch_trace(*tbp, multi_has_constraints(*tbp), ntraces, nops, d_ops, njobs, d_jobs, d_keys, stream);
    if (err) return cuda_fail(err, "esa_trace launch");
    return MAPA_OK;
}

mapa_status mapa_fifo_schedule(int32_t n_devices, int32_t njobs, const int32_t *k, const double *duration,
                               const double *arrival, mapa_trace_op *ops, double *start, double *end) {
    if (njobs < 0 || (njobs > 0 && (!k || !duration || !ops || !start || !end)) || n_devices < 1)
        return fail(MAPA_E_INVALID_ARG, "bad schedule arguments");
    for (int j = 0; j < njobs; ++j) {
        if (k[j] < 1 || k[j] > n_devices) return fail(MAPA_E_INVALID_ARG, "job " + std::to_string(j) + " larger than the machine");
        if (duration[j] < 0 || (arrival && arrival[j] < 0)) return fail(MAPA_E_INVALID_ARG, "negative time");
    }
    // strict FIFO event loop: finishes at time t first (job order), then the
    // head starts while it has arrived and fits; time jumps to the next
    // finish or the head's arrival
    std::vector<std::pair<double, int>> running;  // (end, job)
    int free = n_devices, q = 0, no = 0;
    double t = 0.0;
    while (q < njobs || !running.empty()) {
        std::vector<int> done;
        for (auto &r : running)
            if (r.first <= t) done.push_back(r.second);
        std::sort(done.begin(), done.end());
        for (int j : done) {
            ops[no++] = {1, j};
            free += k[j];
        }
        running.erase(std::remove_if(running.begin(), running.end(),
                                     [t](const std::pair<double, int> &r) { return r.first <= t; }),
                      running.end());
        while (q < njobs && (!arrival || arrival[q] <= t) && k[q] <= free) {
            ops[no++] = {0, q};
            start[q] = t;
            end[q] = t + duration[q];
            free -= k[q];
            running.push_back({end[q], q});
            ++q;
        }
        double nxt = 1e300;
        for (auto &r : running) nxt = std::min(nxt, r.first);
        if (q < njobs && arrival && arrival[q] > t) nxt = std::min(nxt, arrival[q]);
        if (nxt == 1e300) break;
        t = nxt;
    }
    if (q != njobs || no != 2 * njobs) return fail(MAPA_E_INTERNAL, "schedule did not drain");
    return MAPA_OK;
}

mapa_status mapa_simulate(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats, int32_t njobs,
                          const mapa_job *jobs, int32_t policy, uint32_t flags, void *stream, mapa_job_log *out) {
    const NvtxRange nvtx_range_("mapa_simulate");
    if (!t || !pats || njobs < 0 || (njobs > 0 && (!jobs || !out))) return fail(MAPA_E_INVALID_ARG, "null argument");
    if (policy < MAPA_POLICY_BASELINE || policy > MAPA_POLICY_PRESERVE) return fail(MAPA_E_INVALID_ARG, "bad policy");
    if (njobs == 0) return MAPA_OK;
    std::vector<int32_t> kk(njobs);
    std::vector<double> dur(njobs), arr(njobs), st(njobs), en(njobs);
    for (int j = 0; j < njobs; ++j) {
        if (jobs[j].pattern < 0 || jobs[j].pattern >= npats || !pats[jobs[j].pattern])
            return fail(MAPA_E_INVALID_ARG, "job pattern index out of range");
        kk[j] = pats[jobs[j].pattern]->k;
        dur[j] = jobs[j].duration;
        arr[j] = jobs[j].arrival;
    }
    std::vector<mapa_trace_op> ops(2 * (size_t)njobs);
    mapa_status s = mapa_fifo_schedule(t->n, njobs, kk.data(), dur.data(), arr.data(), ops.data(), st.data(), en.data());
    if (s != MAPA_OK) return s;
    static const int32_t kSel[4] = {MAPA_SEL_BASELINE, MAPA_SEL_TOPO, MAPA_SEL_GREEDY, MAPA_SEL_PRESERVE};
    std::vector<mapa_query> q(njobs);
    for (int j = 0; j < njobs; ++j) {
        q[j].busy = 0;
        q[j].pattern = (uint32_t)jobs[j].pattern;
        q[j].selector = kSel[policy];
        q[j].sensitive = policy == MAPA_POLICY_PRESERVE ? (jobs[j].sensitive != 0) : 0;
    }
    cudaStream_t cs = (cudaStream_t)stream;
    void *d_ops = nullptr, *d_jobs = nullptr, *d_keys = nullptr;
    int err;
    const size_t bo = ops.size() * sizeof(mapa_trace_op), bj = q.size() * sizeof(mapa_query), bk = njobs * sizeof(uint64_t);
    if ((err = (int)cudaMalloc(&d_ops, bo + bj + bk))) return cuda_fail(err, "cudaMalloc (simulate)");
    d_jobs = (char *)d_ops + bo;
    d_keys = (char *)d_jobs + bj;
    std::vector<uint64_t> keys(njobs);
    auto cleanup = [&]() { cudaFree(d_ops); };
    if ((err = (int)cudaMemcpyAsync(d_ops, ops.data(), bo, cudaMemcpyHostToDevice, cs)) ||
        (err = (int)cudaMemcpyAsync(d_jobs, q.data(), bj, cudaMemcpyHostToDevice, cs))) {
        cleanup();
        return cuda_fail(err, "H2D (simulate)");
    }
    s = mapa_trace_replay(t, pats, npats, 1, 2 * njobs, (const mapa_trace_op *)d_ops, njobs,
                          (const mapa_query *)d_jobs, (uint64_t *)d_keys, flags & MAPA_F_RAW, stream);
    if (s != MAPA_OK) { cleanup(); return s; }
    if ((err = (int)cudaMemcpyAsync(keys.data(), d_keys, bk, cudaMemcpyDeviceToHost, cs)) ||
        (err = (int)cudaStreamSynchronize(cs))) {
        cleanup();
        return cuda_fail(err, "D2H (simulate)");
    }
    cleanup();
    // host replay of the op order: the busy mask at each ALLOC decodes its key
    std::vector<mapa_decision> dec(njobs);
    s = mapa_decode_trace(t, pats, npats, 2 * njobs, ops.data(), njobs, q.data(), keys.data(), flags & MAPA_F_RAW,
                          dec.data());
    if (s != MAPA_OK) return s;
    for (int j = 0; j < njobs; ++j) {
        const mapa_decision &d = dec[j];
        if (d.status != MAPA_OK) return fail(MAPA_E_INTERNAL, "admitted job without a decision");
        const mapa_pattern *p = pats[jobs[j].pattern];
        mapa_job_log &L = out[j];
        std::memset(&L, 0, sizeof(L));
        L.job = j;
        L.k = p->k;
        L.device_mask = (uint32_t)d.device_mask;
        L.x = d.x; L.y = d.y; L.z = d.z;
        L.agg_bw = d.agg_bw;
        L.preserved_bw = d.preserved_bw;
        L.pred_effbw = d.pred_effbw;
        L.arrival = arr[j];
        L.start = st[j];
        L.end = en[j];
        L.wait = st[j] - arr[j];
    }
    return MAPA_OK;
}

mapa_status mapa_decode_trace(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats, int32_t nops,
                              const mapa_trace_op *ops, int32_t njobs, const mapa_query *jobs, const uint64_t *keys,
                              uint32_t flags, mapa_decision *out) {
    if (!t || !pats || npats < 1 || nops < 0 || njobs < 0 || (nops > 0 && !ops) ||
        (njobs > 0 && (!jobs || !keys || !out)))
        return fail(MAPA_E_INVALID_ARG, "bad decode_trace arguments");
    for (int j = 0; j < njobs; ++j)
        if (jobs[j].pattern >= (uint32_t)npats || !pats[jobs[j].pattern])
            return fail(MAPA_E_INVALID_ARG, "job " + std::to_string(j) + ": pattern index out of range");
    std::vector<mapa_decision> dec(njobs);
    for (auto &d : dec) {
        std::memset(&d, 0, sizeof(d));
        d.status = MAPA_NO_CAPACITY;
    }
    // replay the op order (§3.6): an ALLOC decodes its key on the
    // busy mask of that moment, then claims the devices; RELEASE frees them
    uint64_t busy = 0;
    std::vector<uint64_t> held(njobs, 0);
    std::vector<char> seen(njobs, 0);
    for (int i = 0; i < nops; ++i) {
        const int j = ops[i].job;
        if (j < 0 || j >= njobs || (ops[i].op != 0 && ops[i].op != 1))
            return fail(MAPA_E_INVALID_ARG, "op " + std::to_string(i) + " out of range");
        if (ops[i].op == 1) {
            busy &= ~held[j];
            held[j] = 0;
            continue;
        }
        if (seen[j]) return fail(MAPA_E_INVALID_ARG, "job " + std::to_string(j) + " allocated twice");
        seen[j] = 1;
        const mapa_pattern *p = pats[jobs[j].pattern];
        const int nf = __builtin_popcountll(~busy & nmask_of(t->n));
        mapa_decision &d = dec[j];
        d.k = p->k;
        d.m = p->m;
        if (keys[j] == 0) continue;  // no capacity: state unchanged
        // Topo-aware lays the pattern on its set like Baseline (reading A21)
        const int sel = jobs[j].selector == MAPA_SEL_TOPO ? MAPA_SEL_BASELINE : jobs[j].selector;
        mapa_record rec;
        std::memset(&rec, 0, sizeof(rec));
        rec.key = keys[j];
        mapa_status s = decode_record(t, p, busy, sel, jobs[j].sensitive, flags & MAPA_F_RAW, &rec, &d);
        if (s != MAPA_OK) return s == MAPA_NO_CAPACITY ? fail(MAPA_E_INTERNAL, "nonzero key decoded as no capacity") : s;
        if (d.device_mask & busy) return fail(MAPA_E_INTERNAL, "job " + std::to_string(j) + ": decision overlaps busy devices");
        // the trace kernel does not count leaves: the totals are the closed forms
        d.raw_embeddings = perm_count(nf, p->k);
        d.distinct_matches = d.raw_embeddings / (uint64_t)p->aut;
        d.leaves_scored = 0;
        held[j] = d.device_mask;
        busy |= d.device_mask;
    }
    std::memcpy(out, dec.data(), sizeof(mapa_decision) * (size_t)njobs);
    return MAPA_OK;
}

mapa_status mapa_shard_queries(const mapa_topology *t, const mapa_pattern *const *pats, int32_t npats, int64_t nq,
                               const mapa_query *queries, uint32_t flags, int32_t world, int32_t *owner,
                               double *load) {
    if (!t || !pats || npats < 1 || nq < 0 || world < 1 || (nq > 0 && (!queries || !owner)))
        return fail(MAPA_E_INVALID_ARG, "bad shard arguments");
    // work of a query = the leaves its launch scores: P(|F|, k) in RAW mode,
    // P(|F|, k) / |Aut(P)| canonical (orbit theorem); 0 without capacity
    std::vector<std::pair<double, int64_t>> wq((size_t)nq);
    for (int64_t i = 0; i < nq; ++i) {
        const mapa_query &q = queries[i];
        if (q.pattern >= (uint32_t)npats || !pats[q.pattern])
            return fail(MAPA_E_INVALID_ARG, "query " + std::to_string(i) + ": pattern index out of range");
        const mapa_pattern *p = pats[q.pattern];
        const int nf = __builtin_popcountll(~(uint64_t)q.busy & nmask_of(t->n));
        double w = 0.0;
        if (p->k <= nf) {
            w = 1.0;
            for (int j = 0; j < p->k; ++j) w *= (double)(nf - j);
            if (!(flags & MAPA_F_RAW)) w /= (double)p->aut;
        }
        wq[(size_t)i] = {w, i};
    }
    // LPT: heaviest first (ties by query index), each to the least-loaded rank
    // (ties by rank id): deterministic, max load <= mean + the largest query
    std::stable_sort(wq.begin(), wq.end(), [](const std::pair<double, int64_t> &a, const std::pair<double, int64_t> &b) {
        return a.first > b.first;
    });
    std::vector<double> ld((size_t)world, 0.0);
    for (const auto &x : wq) {
        int r = 0;
        for (int j = 1; j < world; ++j)
            if (ld[(size_t)j] < ld[(size_t)r]) r = j;
        owner[x.second] = r;
        ld[(size_t)r] += x.first;
    }
    if (load)
        for (int j = 0; j < world; ++j) load[j] = ld[(size_t)j];
    return MAPA_OK;
}

mapa_status mapa_quantiles(const double *v, int32_t n, double *out) {
    if (!v || !out || n < 1) return fail(MAPA_E_INVALID_ARG, "quantiles of an empty set");
    std::vector<double> a(v, v + n);
    std::sort(a.begin(), a.end());
    const double ps[5] = {0.0, 0.25, 0.5, 0.75, 1.0};
    for (int i = 0; i < 5; ++i) {
        const double h = ps[i] * (n - 1);
        const int lo = (int)std::floor(h);
        const int hi = std::min(lo + 1, n - 1);
        out[i] = a[lo] + (h - lo) * (a[hi] - a[lo]);
    }
    return MAPA_OK;
}

double mapa_pred_effbw_theta(const double *theta, int32_t x, int32_t y, int32_t z) {
    return eq2_theta(theta ? theta : kTheta, x, y, z);
}

mapa_status mapa_fit_effbw(int32_t n, const int32_t *census, const double *bw, double *theta, double *diag) {
    if (!census || !bw || !theta) return fail(MAPA_E_INVALID_ARG, "null argument");
    if (n < 14) return fail(MAPA_E_INVALID_ARG, "fit_effbw: " + std::to_string(n) + " samples < 14 coefficients (underdetermined)");
    for (int i = 0; i < 3 * n; ++i)
        if (census[i] < 0) return fail(MAPA_E_INVALID_ARG, "fit_effbw: negative census");
    // least squares by Householder QR of the n x 14 feature matrix (column major)
    const int c = 14;
    std::vector<double> A((size_t)n * c), b(bw, bw + n);
    for (int i = 0; i < n; ++i) {
        double f[14];
        eq2_features(census[3 * i], census[3 * i + 1], census[3 * i + 2], f);
        for (int j = 0; j < c; ++j) A[(size_t)j * n + i] = f[j];
    }
    double colmax = 0.0;
    for (double v : A) colmax = std::max(colmax, std::fabs(v));
    std::vector<double> rdiag(c);
    for (int j = 0; j < c; ++j) {
        double *a = &A[(size_t)j * n];
        double nrm = 0.0;
        for (int i = j; i < n; ++i) nrm += a[i] * a[i];
        nrm = std::sqrt(nrm);
        if (nrm <= 1e-12 * std::max(1.0, colmax))
            return fail(MAPA_E_INVALID_ARG, "fit_effbw: rank-deficient feature matrix (feature " + std::to_string(j + 1) +
                                                " is a combination of the others on these censuses)");
        const double alpha = a[j] > 0 ? -nrm : nrm;
        a[j] -= alpha;
        double vv = 0.0;
        for (int i = j; i < n; ++i) vv += a[i] * a[i];
        for (int k = j + 1; k < c; ++k) {
            double *ak = &A[(size_t)k * n];
            double d = 0.0;
            for (int i = j; i < n; ++i) d += a[i] * ak[i];
            const double s2 = 2.0 * d / vv;
            for (int i = j; i < n; ++i) ak[i] -= s2 * a[i];
        }
        double d = 0.0;
        for (int i = j; i < n; ++i) d += a[i] * b[i];
        const double s2 = 2.0 * d / vv;
        for (int i = j; i < n; ++i) b[i] -= s2 * a[i];
        rdiag[j] = alpha;
    }
    double rmin = 1e300, rmax = 0.0;
    for (int j = 0; j < c; ++j) { rmin = std::min(rmin, std::fabs(rdiag[j])); rmax = std::max(rmax, std::fabs(rdiag[j])); }
    for (int j = c - 1; j >= 0; --j) {  // back substitution, R above the diagonal in A
        double v = b[j];
        for (int k = j + 1; k < c; ++k) v -= A[(size_t)k * n + j] * theta[k];
        theta[j] = v / rdiag[j];
    }
    if (diag) {  // relative error ||r|| / ||bw||, RMSE, MAE, condition estimate of R
        double r2 = 0.0, b2 = 0.0, ab = 0.0;
        for (int i = 0; i < n; ++i) {
            const double r = eq2_theta(theta, census[3 * i], census[3 * i + 1], census[3 * i + 2]) - bw[i];
            r2 += r * r;
            ab += std::fabs(r);
            b2 += bw[i] * bw[i];
        }
        diag[0] = b2 > 0 ? std::sqrt(r2 / b2) : 0.0;
        diag[1] = std::sqrt(r2 / n);
        diag[2] = ab / n;
        diag[3] = rmax / rmin;
    }
    return MAPA_OK;
}

mapa_status mapa_pattern_set_effbw_model(mapa_pattern *p, const double *theta) {
    if (!p || !theta) return fail(MAPA_E_INVALID_ARG, "null argument");
    std::memcpy(p->theta, theta, sizeof(p->theta));
    p->lut = rank_table(p->m, p->theta);
    p->uid = next_uid();  // cached allocate graphs baked the old table
    free_luts(p);
    return MAPA_OK;
}

}  // extern "C"
