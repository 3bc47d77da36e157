"""Seeded synthetic workload generators shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the MAPA method (no enumeration, no scores,
no selection).  It only draws inputs: topology description texts, occupancy
(busy) masks, pattern choices, job traces and query lists.  Both the CUDA path
and the CPU oracle consume what it produces; neither side's arithmetic lives
here (task rule: "only the seeded input generators serve both").

Randomness: splitmix64 (Steele et al. 2014), a counter-based generator: the
i-th draw of a stream with seed s is ``mix(s + (i+1) * GOLDEN)``, so any
consumer can regenerate any draw.  Master seed 2110.

Recipes follow SURVEY.md §8(d) "Concrete synthetic inputs" and BASELINE.json
``configs``:

* C1  dgx1v, ring-3, all free.
* C2  dgx1p and summit, 1000-job trace, k in U{2..5}, shape in U{ring,tree,full},
      network in U(6) -> sensitivity + duration, all arrive at
      t=0, strict FIFO, finish-before-allocate.
* C3  cubemesh16, {ring,tree,full} x k in {4,6,8}, busy count b in U{0..16-k},
      uniform busy subset.
* C4  het32 (4 dgx1v islands + SingleNVLink1 ring bridges, rest PCIe) and
      rand32(seed) (i.i.d. classes with probabilities 0.1/0.1/0.1/0.7), full-6,
      all free.
* C5  1e5 queries per topology (cubemesh16, het32): k in U{2..5},
      shape in U{ring,tree,full}, b in U{0..N-k}, selector in U{GREEDY,SENS,INSENS}.
"""
from __future__ import annotations

MASTER_SEED = 2110
_GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1

# Link class names of the topology text format; bandwidths are
# NOT defined here (that is method data: Table 1).
CLASS_NAMES = ("nv2x2", "nv2x1", "nv1x1", "pcie")

SHAPES = ("ring", "tree", "ringtree", "full")

# Selector codes shared by the C-ABI and the oracle's entry points.
SEL_GREEDY, SEL_PRESERVE, SEL_BASELINE = 0, 1, 2


def _mix(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Rng:
    """splitmix64 stream: draw i of seed s = mix(s + (i+1)*golden)."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def u64(self) -> int:
        self.state = (self.state + _GOLDEN) & _M64
        return _mix(self.state)

    def below(self, n: int) -> int:
        """Uniform integer in [0, n) by 64x64->128 multiply-shift (bias < 2^-50)."""
        if n <= 0:
            raise ValueError("n must be positive")
        return (self.u64() * n) >> 64

    def randint(self, lo: int, hi: int) -> int:
        """Uniform integer in [lo, hi] (inclusive)."""
        return lo + self.below(hi - lo + 1)

    def choice(self, seq):
        return seq[self.below(len(seq))]

    def subset(self, n: int, b: int) -> list[int]:
        """Uniform b-subset of range(n), by partial Fisher-Yates."""
        a = list(range(n))
        for i in range(b):
            j = i + self.below(n - i)
            a[i], a[j] = a[j], a[i]
        return sorted(a[:b])


def stream(seed: int, index: int) -> Rng:
    """Per-item stream: seed XOR index."""
    return Rng((seed ^ index) & _M64)


# ---------------------------------------------------------------------------
# Topology texts (format: SPEC S:115 field names; syntax documented in DESIGN.md)
#   name <str>
#   devices <n>
#   sockets <id,id,...> <id,...> ...
#   link <a> <b> <class>        (1-based ids, class in CLASS_NAMES)
# Unlisted pairs are PCIe.
# ---------------------------------------------------------------------------

# dgx1v cube-mesh wiring of SPEC S:46 (1-based), used as the island of het32.
_DGX_DOUBLE = [(1, 4), (1, 5), (2, 3), (2, 6), (3, 4), (5, 8), (6, 7), (7, 8)]
_DGX_SINGLE = [(1, 2), (1, 3), (2, 4), (3, 7), (4, 8), (5, 6), (5, 7), (6, 8)]


def topology_text(name: str, n: int, sockets: list[list[int]],
                  links: list[tuple[int, int, str]]) -> str:
    lines = [f"name {name}", f"devices {n}",
             "sockets " + " ".join(",".join(str(d) for d in s) for s in sockets)]
    for a, b, c in links:
        lines.append(f"link {a} {b} {c}")
    return "\n".join(lines) + "\n"


def het32_text() -> str:
    """het32: 4 dgx1v islands, ids 8i+1..8i+8 with SPEC S:46
    edges shifted; bridges (8i+j)<->(8((i+1) mod 4)+j), j=1..8, SingleNVLink1;
    every other pair PCIe.  Sockets = the 4 islands."""
    links = []
    for i in range(4):
        o = 8 * i
        links += [(a + o, b + o, "nv2x2") for a, b in _DGX_DOUBLE]
        links += [(a + o, b + o, "nv2x1") for a, b in _DGX_SINGLE]
    for i in range(4):
        for j in range(1, 9):
            a, b = 8 * i + j, 8 * ((i + 1) % 4) + j
            links.append((min(a, b), max(a, b), "nv1x1"))
    sockets = [list(range(8 * i + 1, 8 * i + 9)) for i in range(4)]
    return topology_text("het32", 32, sockets, links)


def het64_text() -> str:
    """het64 (servers beyond 32 accelerators): het32's
    construction with 8 dgx1v islands, ids 8i+1..8i+8; bridges
    (8i+j)<->(8((i+1) mod 8)+j) SingleNVLink1; sockets = the 8 islands."""
    links = []
    for i in range(8):
        o = 8 * i
        links += [(a + o, b + o, "nv2x2") for a, b in _DGX_DOUBLE]
        links += [(a + o, b + o, "nv2x1") for a, b in _DGX_SINGLE]
    for i in range(8):
        for j in range(1, 9):
            a, b = 8 * i + j, 8 * ((i + 1) % 8) + j
            links.append((min(a, b), max(a, b), "nv1x1"))
    sockets = [list(range(8 * i + 1, 8 * i + 9)) for i in range(8)]
    return topology_text("het64", 64, sockets, links)


def rand_text(n: int, seed: int, probs=(0.1, 0.1, 0.1, 0.7)) -> str:
    """randN(seed): every pair i.i.d. class with the given probabilities
    (nv2x2, nv2x1, nv1x1, pcie).  Pair (a,b), a<b, uses stream(seed, a*64+b)."""
    cum = []
    acc = 0.0
    for p in probs:
        acc += p
        cum.append(acc)
    links = []
    for a in range(1, n + 1):
        for b in range(a + 1, n + 1):
            u = stream(seed, a * 64 + b).u64() / 2.0 ** 64
            c = next(i for i, t in enumerate(cum) if u < t or i == 3)
            if c != 3:
                links.append((a, b, CLASS_NAMES[c]))
    half = n // 2
    sockets = [list(range(1, half + 1)), list(range(half + 1, n + 1))]
    return topology_text(f"rand{n}_{seed}", n, sockets, links)


# ---------------------------------------------------------------------------
# Occupancy masks, patterns, queries
# ---------------------------------------------------------------------------

def busy_mask(rng: Rng, n: int, k: int) -> int:
    """b in U{0..n-k} busy devices, uniform b-subset (C3/C5 recipe); 0-based bits."""
    b = rng.randint(0, n - k)
    m = 0
    for d in rng.subset(n, b):
        m |= 1 << d
    return m


def c3_queries(seed: int = MASTER_SEED, per_case: int = 1000, n: int = 16):
    """C3: for shape in {ring,tree,full} x k in {4,6,8}: per_case queries
    (shape, k, busy, selector, sensitive)."""
    out = []
    idx = 0
    for shape in ("ring", "tree", "full"):
        for k in (4, 6, 8):
            for _ in range(per_case):
                r = stream(seed, idx)
                idx += 1
                busy = busy_mask(r, n, k)
                sel = r.below(3)  # 0 GREEDY, 1 SENS, 2 INSENS
                out.append(_query(shape, k, busy, sel))
    return out


def _query(shape, k, busy, sel3):
    if sel3 == 0:
        return dict(shape=shape, k=k, busy=busy, selector=SEL_GREEDY, sensitive=0)
    if sel3 == 1:
        return dict(shape=shape, k=k, busy=busy, selector=SEL_PRESERVE, sensitive=1)
    return dict(shape=shape, k=k, busy=busy, selector=SEL_PRESERVE, sensitive=0)


def c5_queries(n: int, count: int = 100_000, seed: int = MASTER_SEED):
    """C5: k in U{2..5}, shape in U{ring,tree,full}, busy b in U{0..n-k},
    selector in U{GREEDY, SENS, INSENS}.  Query i uses stream(seed+n, i)."""
    out = []
    for i in range(count):
        r = stream(seed + n, i)
        k = r.randint(2, 5)
        shape = ("ring", "tree", "full")[r.below(3)]
        busy = busy_mask(r, n, k)
        out.append(_query(shape, k, busy, r.below(3)))
    return out


# ---------------------------------------------------------------------------
# Job traces (C2).  Network mix and durations: SPEC S:177-178 (sensitivity
# labels per P:767 / Fig. 6b).
# ---------------------------------------------------------------------------

NETWORKS = (("alexnet", True, 511), ("vgg16", True, 785), ("resnet50", True, 600),
            ("inceptionv3", True, 650), ("caffenet", False, 300), ("googlenet", False, 350))

OP_ALLOC, OP_RELEASE = 0, 1


def c2_jobs(seed: int, count: int = 1000):
    """1000 jobs: network U(6) -> (sensitive, duration); k U{2..5}; shape U{ring,tree,full}."""
    jobs = []
    for j in range(count):
        r = stream(seed, j)
        name, sens, dur = NETWORKS[r.below(6)]
        k = r.randint(2, 5)
        shape = ("ring", "tree", "full")[r.below(3)]
        jobs.append(dict(job=j, network=name, sensitive=int(sens), duration=dur, k=k, shape=shape))
    return jobs


def sim_jobs(seed: int, count: int = 300, kmax: int = 5):
    """Simulator job file (§4 "Jobs configuration"): network U(6)
    -> (sensitive, duration), requested GPUs k U{1..kmax},
    pattern shape U{ring, tree, full} (k = 1: the singleton), all at t = 0."""
    jobs = []
    for j in range(count):
        r = stream(seed ^ 0x5117, j)
        name, sens, dur = NETWORKS[r.below(6)]
        k = r.randint(1, kmax)
        shape = ("ring", "tree", "full")[r.below(3)] if k > 1 else "full"
        jobs.append(dict(job=j, network=name, sensitive=int(sens), duration=dur, k=k, shape=shape))
    return jobs


def spec_jobs(seed: int, count: int = 300, kmin: int = 1, kmax: int = 5):
    """SPEC generate_jobs (§4 "Jobs configuration"):
    network U(6) -> (sensitive, duration), requested GPUs
    U{kmin..kmax}, shape Ring for k >= 2 (NCCL's all-reduce ring) and the
    singleton for k = 1, all at t = 0.  The job mix of the directional
    simulator checks (SPEC acceptance criteria 6-7)."""
    jobs = []
    for j in range(count):
        r = stream(seed ^ 0x5EC, j)
        name, sens, dur = NETWORKS[r.below(6)]
        k = r.randint(kmin, kmax)
        jobs.append(dict(job=j, network=name, sensitive=int(sens), duration=dur, k=k, shape="ring" if k >= 2 else "full"))
    return jobs


def fifo_ops(jobs, n_devices: int):
    """Op sequence of a strict-FIFO replay where every job arrives at t=0
    (SPEC S:404).  Admission depends only on the FREE COUNT (the
    hardware graph is complete), so the ALLOC/RELEASE order is the same
    for every policy and is computed here without any scoring.  Finish events
    at equal times are processed before allocation attempts, in job order.
    Returns a list of (op, job_index)."""
    ops = []
    free = n_devices
    t = 0
    running = []  # (end_time, job)
    q = 0
    while q < len(jobs) or running:
        while q < len(jobs) and jobs[q]["k"] <= free:
            j = jobs[q]
            ops.append((OP_ALLOC, j["job"]))
            free -= j["k"]
            running.append((t + j["duration"], j["job"]))
            q += 1
        if not running:
            if q < len(jobs):
                raise ValueError("job larger than the machine")
            break
        t = min(e for e, _ in running)
        done = sorted(jb for e, jb in running if e == t)
        running = [(e, jb) for e, jb in running if e != t]
        for jb in done:
            ops.append((OP_RELEASE, jb))
            free += jobs[jb]["k"]
    return ops
