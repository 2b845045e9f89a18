import sys, time
sys.path.insert(0, ".")
import paper_1805_00569_b200 as pk
eng = pk.Engine(0)
for m in (8192, 8192, 4096):
    t = time.time()
    r = eng.probe_potrf(m)
    print(m, round(time.time() - t, 3), "s wall", {k: round(v, 3) for k, v in r.items()})
