"""One pruned Preserve-sensitive ring-16 allocation on torus2d16 (all free) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_03214_b200 as mp
t = mp.Topology("torus2d16")
d = mp.allocate(t, mp.Pattern.make("ring", 16), 1, True, deep=True, prune=True)
print(d["leaves"], d["devices"])
