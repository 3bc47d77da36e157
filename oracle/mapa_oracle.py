"""Pure-Python MAPA oracle (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Every function is the plain definition from the paper, written out, citing the
passage it follows.  Device ids are 0-based here (SPEC's 1-based id - 1; lex
order is unchanged).  No symmetry breaking, no incremental scoring,
no key packing: those belong to the CUDA path and are what this oracle tests.

Readings of the paper where it is silent or garbled (SURVEY.md §8(c) A1-A18,
restated in DESIGN.md):
  A1 tie-break: lex-smallest sorted device tuple, then lex-smallest sorted
     used-edge list; the reported mapping is the lex-first
     permutation of that device tuple producing that edge set.
  A2 matches are deduplicated by (device set, used-edge set).
  A3 Alg. 1 starts from an empty incumbent: the first match always wins.
  A4 census counts the USED edges E(P)∩E(M).
  A5 SingleNVLink1 (20 GB/s) counts toward y.
  A6 Eq. 3 deletes V(M) from the *available* graph (P:711 garble; §3.6).
"""
from __future__ import annotations

import itertools
from fractions import Fraction

# Table 1 "Peak Bandwidths per link": class name -> GB/s.
LINK_BW = {"nv2x2": 50, "nv2x1": 25, "nv1x1": 20, "pcie": 12}
PCIE_BW = 12  # "If two GPUs have no NVLink connectivity ... labeled with ... 12"

# Table 4 "Values of Coefficients", theta_1..theta_14, exact decimals.
THETA = tuple(Fraction(s) for s in (
    "16.396", "4.536", "1.556", "-20.694", "-9.467", "7.615", "-7.973",
    "12.733", "-4.195", "-8.413", "62.851", "27.418", "-5.114", "-46.973"))

GREEDY, PRESERVE, BASELINE = 0, 1, 2


# ---------------------------------------------------------------------------
# Hardware graph (§3.2; SPEC topology module S:17-120)
# ---------------------------------------------------------------------------

class Topology:
    """Complete weighted graph: w[u][v] = highest link bandwidth, PCIe 12 when
    no NVLink."""

    def __init__(self, name: str, n: int, links: dict, sockets=None):
        self.name = name
        self.n = n
        self.sockets = sockets or [list(range(n))]
        self.w = [[0] * n for _ in range(n)]
        for u in range(n):
            for v in range(n):
                if u != v:
                    self.w[u][v] = PCIE_BW
        for (a, b), bw in links.items():
            self.w[a][b] = bw
            self.w[b][a] = bw

    def bw(self, u: int, v: int) -> int:
        """edge_bandwidth: NVLink class BW if linked, else 12."""
        if u == v or not (0 <= u < self.n and 0 <= v < self.n):
            raise ValueError("invalid device pair")
        return self.w[u][v]


def _links(pairs_1based, bw):
    return {(a - 1, b - 1): bw for a, b in pairs_1based}


# SPEC S:46 (dgx1v) -- edge classes fixed by P:261 (1-5 double, 1-2 single,
# 1-6 PCIe) and the §2.2 worked examples ({1,2,5}=87, {1,3,4}=125).
DGX1V_DOUBLE = [(1, 4), (1, 5), (2, 3), (2, 6), (3, 4), (5, 8), (6, 7), (7, 8)]
DGX1V_SINGLE = [(1, 2), (1, 3), (2, 4), (3, 7), (4, 8), (5, 6), (5, 7), (6, 8)]


def builtin(name: str) -> Topology:
    """builtin_topology."""
    if name == "dgx1v":
        links = _links(DGX1V_DOUBLE, 50)
        links.update(_links(DGX1V_SINGLE, 25))
        return Topology(name, 8, links, [[0, 1, 2, 3], [4, 5, 6, 7]])
    if name == "dgx1p":  # same wiring, every NVLink edge SingleNVLink1 (20)
        links = _links(DGX1V_DOUBLE + DGX1V_SINGLE, 20)
        return Topology(name, 8, links, [[0, 1, 2, 3], [4, 5, 6, 7]])
    if name == "summit":  # two DoubleNVLink2 triples, cross-socket PCIe
        links = {}
        for tri in ((0, 1, 2), (3, 4, 5)):
            for a, b in itertools.combinations(tri, 2):
                links[(a, b)] = 50
        return Topology(name, 6, links, [[0, 1, 2], [3, 4, 5]])
    if name == "torus2d16":  # 4x4 wraparound, rows double, columns single
        links = {}
        for r in range(4):
            for c in range(4):
                u = 4 * r + c
                h = 4 * r + (c + 1) % 4
                v = 4 * ((r + 1) % 4) + c
                links[(min(u, h), max(u, h))] = 50
                links[(min(u, v), max(u, v))] = 25
        return Topology(name, 16, links, [list(range(8)), list(range(8, 16))])
    if name == "cubemesh16":  # two dgx1v meshes + 4 SingleNVLink2 bridges
        links = _links(DGX1V_DOUBLE, 50)
        links.update(_links(DGX1V_SINGLE, 25))
        links.update(_links([(a + 8, b + 8) for a, b in DGX1V_DOUBLE], 50))
        links.update(_links([(a + 8, b + 8) for a, b in DGX1V_SINGLE], 25))
        links.update(_links([(1, 9), (4, 12), (5, 13), (8, 16)], 25))
        return Topology(name, 16, links, [list(range(8)), list(range(8, 16))])
    raise ValueError(f"unknown topology {name!r}; valid: dgx1v dgx1p summit torus2d16 cubemesh16")


def parse_topology(text: str) -> Topology:
    """Topology file (SPEC S:115 fields: name, devices, sockets, links; syntax
    in DESIGN.md).  1-based ids in the file."""
    name, n, sockets, links = None, None, None, {}
    for ln, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        f = line.split()
        if f[0] == "name":
            name = f[1]
        elif f[0] == "devices":
            n = int(f[1])
        elif f[0] == "sockets":
            sockets = [[int(x) - 1 for x in s.split(",")] for s in f[1:]]
        elif f[0] == "link":
            a, b, c = int(f[1]) - 1, int(f[2]) - 1, f[3]
            if a == b or not (0 <= a < n and 0 <= b < n):
                raise ValueError(f"line {ln}: bad link")
            key = (min(a, b), max(a, b))
            if key in links:
                raise ValueError(f"line {ln}: duplicate link")
            links[key] = LINK_BW[c]
        else:
            raise ValueError(f"line {ln}: unknown field {f[0]}")
    return Topology(name, n, links, sockets)


def induced_total_bandwidth(topo: Topology, vertices) -> int:
    """sum of w over all unordered pairs within `vertices`."""
    vs = sorted(vertices)
    return sum(topo.bw(u, v) for u, v in itertools.combinations(vs, 2))


# ---------------------------------------------------------------------------
# Application pattern (§3.1, Fig. 4; SPEC make_pattern S:143-151)
# ---------------------------------------------------------------------------

def make_pattern(shape: str, n: int):
    """Returns (k, sorted edge list).  Ring: cycle 0-1-..-(n-1)-0, n=2 a single
    edge; Tree: balanced binary tree, children of i are 2i+1, 2i+2; RingTree:
    union; Full: all pairs; n=1: empty singleton."""
    if n < 1:
        raise ValueError("n >= 1")
    ring = set()
    if shape in ("ring", "ringtree"):
        if n == 1 and shape == "ring":
            raise ValueError("Ring requires n >= 2")
        if n == 2:
            ring = {(0, 1)}
        elif n >= 3:
            ring = {(min(i, (i + 1) % n), max(i, (i + 1) % n)) for i in range(n)}
    tree = set()
    if shape in ("tree", "ringtree"):
        for i in range(n):
            for c in (2 * i + 1, 2 * i + 2):
                if c < n:
                    tree.add((i, c))
    if shape == "ring":
        e = ring
    elif shape == "tree":
        e = tree
    elif shape == "ringtree":
        e = ring | tree
    elif shape == "full":
        e = set(itertools.combinations(range(n), 2))
    elif shape == "edgeless":
        e = set()
    else:
        raise ValueError(f"unknown shape {shape}")
    return n, sorted(e)


def automorphism_count(k: int, edges) -> int:
    """|Aut(P)| by brute force over all k! vertex permutations."""
    es = {frozenset(e) for e in edges}
    c = 0
    for s in itertools.permutations(range(k)):
        if {frozenset((s[a], s[b])) for a, b in edges} == es:
            c += 1
    return c


# ---------------------------------------------------------------------------
# Scores
# ---------------------------------------------------------------------------

def used_edges(mapping, pedges):
    """E(P) ∩ E(M) realised: image of every pattern edge, as a
    sorted list of (lo, hi) device pairs."""
    return sorted((min(mapping[a], mapping[b]), max(mapping[a], mapping[b])) for a, b in pedges)


def aggregated_bw(topo: Topology, E) -> int:
    """Eq. 1: sum of w(e) over the used edges."""
    return sum(topo.bw(u, v) for u, v in E)


def link_census(topo: Topology, E):
    """(x, y, z) = #used edges that are double NVLink (50), single NVLink
    (25 or 20, reading A5), PCIe (12) — §3.4.3."""
    x = y = z = 0
    for u, v in E:
        b = topo.bw(u, v)
        if b == 50:
            x += 1
        elif b in (25, 20):
            y += 1
        elif b == 12:
            z += 1
        else:
            raise ValueError("unknown link bandwidth")
    return x, y, z


def eq2_exact(x: int, y: int, z: int, theta=THETA) -> Fraction:
    """Eq. 2, exact rational with Table 4 theta."""
    t = theta
    one = Fraction(1)
    return (t[0] * x + t[1] * y + t[2] * z
            + t[3] * (one / (x + 1)) + t[4] * (one / (y + 1)) + t[5] * (one / (z + 1))
            + t[6] * (x * y) + t[7] * (y * z) + t[8] * (z * x)
            + t[9] * (one / (x * y + 1)) + t[10] * (one / (y * z + 1)) + t[11] * (one / (z * x + 1))
            + t[12] * (x * y * z) + t[13] * (one / (x * y * z + 1)))


def eq2(x: int, y: int, z: int) -> float:
    """Eq. 2 as a double (reporting value)."""
    return float(eq2_exact(x, y, z))


def preserved_bw(topo: Topology, free, S) -> int:
    """Eq. 3: total bandwidth of the subgraph of the AVAILABLE graph
    induced by the free devices left after removing V(M) (reading A6).  Direct
    double loop over survivor pairs."""
    rest = sorted(set(free) - set(S))
    tot = 0
    for i in range(len(rest)):
        for j in range(i + 1, len(rest)):
            tot += topo.bw(rest[i], rest[j])
    return tot


# ---------------------------------------------------------------------------
# Matching + selection (§3.3, Alg. 1, §4)
# ---------------------------------------------------------------------------

def free_devices(topo: Topology, busy_mask: int):
    return [d for d in range(topo.n) if not (busy_mask >> d) & 1]


def find_matches(topo: Topology, busy_mask: int, k: int, pedges):
    """All matches of P in the available graph, deduplicated by (device set,
    used edges) (reading A2), in lex order of (sorted device tuple, sorted
    used-edge list).  Every injective map is an embedding because G is complete
    (P:491).  Returns (matches, raw) where each match is (S, E, first_mapping)
    and raw counts every injective map."""
    F = free_devices(topo, busy_mask)
    out = []
    raw = 0
    if k > len(F):
        return out, 0
    for S in itertools.combinations(F, k):          # lexicographic
        seen = {}
        for pi in itertools.permutations(S):          # lexicographic => first pi is lex-min
            raw += 1
            E = tuple(used_edges(pi, pedges))
            if E not in seen:
                seen[E] = pi
        for E in sorted(seen):
            out.append((S, list(E), seen[E]))
    return out, raw


def allocate(topo: Topology, busy_mask: int, k: int, pedges, selector: int, sensitive: bool, theta=None):
    """Greedy (argmax AggBW), Preserve (Alg. 1: sensitive -> argmax
    predicted EffBW, insensitive -> argmax PreservedBW) or Baseline
    (constant score => lowest ids).  Strict '>' over the lex-ordered
    match list = Alg. 1's "first wins" loop + SPEC's tie-break (A1, A3)."""
    F = free_devices(topo, busy_mask)
    matches, raw = find_matches(topo, busy_mask, k, pedges)
    if k > len(F):
        return dict(status="no_capacity", raw=0, distinct=0)
    best = None
    for S, E, pi in matches:
        agg = aggregated_bw(topo, E)
        x, y, z = link_census(topo, E)
        eff = eq2_exact(x, y, z) if theta is None else eq2_exact(x, y, z, tuple(Fraction(t) for t in theta))
        pres = preserved_bw(topo, F, S)
        if selector == GREEDY:
            s = agg
        elif selector == PRESERVE:
            s = eff if sensitive else pres
        elif selector == BASELINE:
            s = 0
        else:
            raise ValueError("selector")
        if best is None or s > best[0]:
            best = (s, S, E, pi, agg, (x, y, z), eff, pres)
    s, S, E, pi, agg, cen, eff, pres = best
    return dict(status="ok", devices=tuple(S), mapping=tuple(pi), used_edges=[tuple(e) for e in E],
                x=cen[0], y=cen[1], z=cen[2], agg_bw=agg, preserved_bw=pres,
                pred_effbw=float(eff), pred_effbw_exact=eff,
                raw=raw, distinct=len(matches))


def device_mask(devs) -> int:
    m = 0
    for d in devs:
        m |= 1 << d
    return m


def replay_trace(topo: Topology, jobs, ops, patterns, policy: str, allocate_fn=None):
    """Replays an ALLOC/RELEASE op list (workloads.fifo_ops) with MAPA state
    management (§3.6): allocate removes the chosen devices, release
    adds them back.  policy 'preserve' uses each job's sensitivity (Alg. 1);
    'greedy' uses AggBW.  allocate_fn defaults to allocate() (the C oracle's
    coracle.allocate has the same signature).  Returns {job: decision}."""
    alloc = allocate_fn or allocate
    busy = 0
    held = {}
    out = {}
    for op, j in ops:
        if op == 0:
            job = jobs[j]
            k, pe = patterns[(job["shape"], job["k"])]
            if policy == "preserve":
                d = alloc(topo, busy, k, pe, PRESERVE, bool(job["sensitive"]))
            else:
                d = alloc(topo, busy, k, pe, GREEDY, False)
            if d["status"] != "ok":
                raise RuntimeError("trace admitted a job without capacity")
            m = device_mask(d["devices"])
            assert busy & m == 0
            busy |= m
            held[j] = m
            out[j] = d
        else:
            busy &= ~held.pop(j)
    return out


# ---------------------------------------------------------------------------
# Policies above the path and the simulator (§4; §5 P:871-880;
# SPEC policies S:326-344, simulator S:386-439) -- SURVEY §8(f) NEXT 2.
# ---------------------------------------------------------------------------

def topo_partitions(topo: Topology):
    """Reading A21 of "recursive bi-partitioning ... under the same PCIe tree
    (CPU socket)": every socket group, then each half
    of it (sorted ids, first half = ceil(n/2)), recursively down to single
    devices, plus the whole machine."""
    parts = []

    def rec(g):
        g = sorted(g)
        parts.append(tuple(g))
        if len(g) > 1:
            h = (len(g) + 1) // 2
            rec(g[:h])
            rec(g[h:])

    for g in topo.sockets:
        rec(g)
    parts.append(tuple(range(topo.n)))
    return parts


def select_topo_aware(topo: Topology, busy_mask: int, k: int):
    """SPEC select_topo_aware: the smallest partition with >= k free devices
    (ties: the partition holding the lowest device id), its k lowest free
    ids; no partition fits -> the k lowest free ids (global fallback).
    Returns the device tuple, or None without capacity."""
    free = set(free_devices(topo, busy_mask))
    if len(free) < k:
        return None
    fits = [p for p in topo_partitions(topo) if len([d for d in p if d in free]) >= k]
    if fits:
        best = min(fits, key=lambda p: (len(p), p[0]))
        return tuple(sorted(d for d in best if d in free)[:k])
    return tuple(sorted(free)[:k])


def allocate_policy(topo: Topology, busy_mask: int, k: int, pedges, policy: str, sensitive: bool,
                    allocate_fn=None):
    """One decision of the evaluation's four policies.  Baseline
    and Topo-aware choose the device set by their rule; the job's pattern is
    then laid on it by the same tie-break as every policy (lex-smallest used
    edge list), i.e. the Baseline allocation restricted to that set."""
    alloc = allocate_fn or allocate
    if policy == "greedy":
        return alloc(topo, busy_mask, k, pedges, GREEDY, False)
    if policy == "preserve":
        return alloc(topo, busy_mask, k, pedges, PRESERVE, sensitive)
    if policy == "baseline":
        S = tuple(free_devices(topo, busy_mask)[:k]) if len(free_devices(topo, busy_mask)) >= k else None
    elif policy == "topo":
        S = select_topo_aware(topo, busy_mask, k)
    else:
        raise ValueError(policy)
    if S is None:
        return dict(status="no_capacity")
    only = ((1 << topo.n) - 1) & ~device_mask(S)
    d = alloc(topo, only, k, pedges, BASELINE, False)
    # Eq. 3 is scored on the free set at allocation time, not on S alone
    d = dict(d)
    d["preserved_bw"] = preserved_bw(topo, free_devices(topo, busy_mask), S)
    return d


def simulate(topo: Topology, jobs, policy: str, allocate_fn=None):
    """SPEC run_simulation, written as the paper's cycle of
    events: all jobs wait in a FIFO queue (arrival times, default
    0); at every event time, first the jobs whose execution time has elapsed
    release their GPUs (job order), then the queue head is allocated while it
    has arrived and enough GPUs are free.  jobs: dicts with k, edges
    (pattern), sensitive, duration[, arrival].  Returns one log dict per job
    (job order): devices, census, agg_bw, pred_effbw, preserved_bw at
    allocation, arrival, start, end, wait."""
    for j in jobs:
        if j["k"] > topo.n:
            raise ValueError("job larger than the machine")
    busy = 0
    t = 0.0
    queue = list(range(len(jobs)))
    running = {}  # job -> (end, mask)
    log = {}
    while queue or running:
        for j in sorted(j for j, (e, _) in running.items() if e <= t):
            busy &= ~running.pop(j)[1]
        while queue:
            j = queue[0]
            job = jobs[j]
            arr = job.get("arrival", 0.0)
            if arr > t or job["k"] > topo.n - bin(busy).count("1"):
                break
            d = allocate_policy(topo, busy, job["k"], job["edges"], policy, bool(job["sensitive"]), allocate_fn)
            m = device_mask(d["devices"])
            assert d["status"] == "ok" and busy & m == 0
            busy |= m
            running[j] = (t + job["duration"], m)
            log[j] = dict(job=j, k=job["k"], devices=tuple(d["devices"]), x=d["x"], y=d["y"], z=d["z"],
                          agg_bw=d["agg_bw"], preserved_bw=d["preserved_bw"], pred_effbw=float(d["pred_effbw"]),
                          arrival=arr, start=t, end=t + job["duration"], wait=t - arr)
            queue.pop(0)
        nxt = [e for e, _ in running.values()]
        if queue and jobs[queue[0]].get("arrival", 0.0) > t:
            nxt.append(jobs[queue[0]]["arrival"])
        if not nxt:
            break
        t = min(nxt)
    return [log[j] for j in range(len(jobs))]


def quantiles7(values):
    """min, 25th, 50th, 75th percentile, max by linear interpolation between
    order statistics (SPEC summarize_log S:427-431, "type 7")."""
    v = sorted(values)
    if not v:
        raise ValueError("empty")
    out = []
    for p in (0.0, 0.25, 0.5, 0.75, 1.0):
        h = p * (len(v) - 1)
        lo = int(h)
        hi = min(lo + 1, len(v) - 1)
        out.append(v[lo] + (h - lo) * (v[hi] - v[lo]))
    return tuple(out)


# ---------------------------------------------------------------------------
# Eq. 2 regression (§3.4.3; SPEC fit_effbw_model S:286-294)
# ---------------------------------------------------------------------------

def eq2_features(x: int, y: int, z: int):
    """The 14 terms of Eq. 2 in theta order; the model is linear in theta."""
    return [x, y, z, 1 / (x + 1), 1 / (y + 1), 1 / (z + 1), x * y, y * z, z * x,
            1 / (x * y + 1), 1 / (y * z + 1), 1 / (z * x + 1), x * y * z, 1 / (x * y * z + 1)]


def fit_effbw(samples):
    """Ordinary least squares over the 14 features (numpy.linalg.lstsq as the
    library primitive).  samples: [(x, y, z, bw)].  Returns (theta, rel_err)
    with rel_err = ||residual|| / ||bw|| (reading A23)."""
    import numpy as np
    if len(samples) < 14:
        raise ValueError("underdetermined: fewer than 14 samples")
    A = np.array([eq2_features(*s[:3]) for s in samples], dtype=np.float64)
    b = np.array([s[3] for s in samples], dtype=np.float64)
    theta, _res, rank, _sv = np.linalg.lstsq(A, b, rcond=None)
    if rank < 14:
        raise ValueError("rank-deficient feature matrix")
    r = A @ theta - b
    return [float(t) for t in theta], float(np.linalg.norm(r) / np.linalg.norm(b))
